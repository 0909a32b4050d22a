"""Multi-GPU round through the C-ABI, checked against the oracle (needs >= 2 GPUs).

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 scripts/dist_round_check.py

One process per GPU: every rank computes the same placement (push placement), trains
its share, fl_aggregate runs k_fedavg4<false> -> ncclAllReduce([S_g ‖ N_g]) -> k_finalize
(P:330), and every rank must hold the same θ_new.  Rank 0 compares θ_new with the
fp64 oracle's whole round (1e-3, reading A21) and prints the round stats (max-over-ranks
round time and "timedelta workers").  Four queued rounds with changing cohorts
(stats off) exercise the asynchronous path first.
"""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2306_17453_b200 as fl  # noqa: E402
import synth  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    dist.init_process_group("gloo")
    torch.cuda.set_device(local)
    obj = [fl.fl_nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    wl = synth.preset("C2", n_pop=24, n_cohort=24)
    sizes = np.minimum(synth.client_sizes(wl), 200)
    _, x, y = synth.population(wl, sizes)
    theta = synth.init_params("cnn")
    cfg = fl.Config(model="cnn", batch_size=wl.B, local_epochs=wl.E, lr=wl.lr, rank=rank, world_size=world,
                    device=local, nccl_unique_id=obj[0])
    ctx = fl.fl_round_init(cfg, sizes, torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), theta)
    rng = np.random.default_rng(4)
    cohorts = [rng.choice(24, size=k, replace=False) for k in (24, 5, 13, 9)]
    th = theta
    for r, c in enumerate(cohorts):
        ctx.fl_round(c, round_index=r, stats=False)
    st = ctx.fl_get_stats()
    out = ctx.fl_get_global_params()
    allout = [None] * world
    dist.all_gather_object(allout, out.tobytes())
    assert all(o == allout[0] for o in allout), "ranks hold different θ_new"
    if rank == 0:
        for r, c in enumerate(cohorts):
            th, _, _ = oracle.fedavg_round("cnn", th.astype(np.float32), x, y, sizes, c, wl.B, wl.E, wl.lr, rnd=r)
        err = float(np.max(np.abs(out - th)))
        print(f"[dist_round_check] world {world}: max|gpu-oracle| after 4 rounds = {err:.2e}; stats {st}")
        assert err <= 1e-3, err
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
