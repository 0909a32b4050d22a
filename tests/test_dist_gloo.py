"""Multi-rank host logic on CPU (world size 2, gloo) — the N > 1 path minus the GPU.

Every rank computes the placement with the library's own host planner
(fl_place_plan); the plans must be identical on all ranks (push placement needs no
message), the local shares must partition the cohort, and the per-rank partial
aggregates [S_g ‖ N_g] summed by an allreduce must reproduce the flat FedAvg of the
whole cohort (Eq. 1-2 associativity) — the same decomposition fl_aggregate
performs with NCCL.  Client models come from the oracle (test infrastructure).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import paper_2306_17453_b200 as fl
import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        wl = synth.preset("C1", n_pop=40, n_cohort=23)
        sizes = synth.client_sizes(wl)
        cohort = synth.cohort(wl)
        ids, off = fl.fl_place_plan("bu", cohort, sizes, wl.B, world)
        plans = [None] * world
        dist.all_gather_object(plans, (ids.tolist(), off.tolist()))
        assert all(p == plans[0] for p in plans), "plans differ across ranks"
        local = ids[off[rank]:off[rank + 1]]
        # this rank's clients, trained by the oracle from θ_g
        _, x, y = synth.population(wl, sizes)
        pop_off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        theta = synth.init_params("logreg").astype(np.float64)
        tk, _ = oracle.train_clients("logreg", theta, x, y, pop_off, local, wl.B, wl.E, wl.lr, threads=1)
        n = sizes[local].astype(np.float64)
        S = (n[:, None] * (tk - theta[None, :])).sum(0) if len(local) else np.zeros_like(theta)
        buf = torch.from_numpy(np.concatenate([S, [n.sum()]]))
        dist.all_reduce(buf)  # what fl_aggregate does with ncclAllReduce (fp64 sum)
        out = theta + buf[:-1].numpy() / buf[-1].item()
        shares = [None] * world
        dist.all_gather_object(shares, sorted(local.tolist()))
        if rank == 0:
            allc = sorted(sum(shares, []))
            assert allc == sorted(cohort.tolist()), "shares do not partition the cohort"
            tk_all, _ = oracle.train_clients("logreg", theta, x, y, pop_off, cohort, wl.B, wl.E, wl.lr, threads=1)
            ref, N = oracle.fedavg(tk_all, sizes[cohort])
            assert N == buf[-1].item()
            assert np.max(np.abs(out - ref)) < 1e-12
        q.put((rank, "ok"))
    except Exception as e:  # report to the parent
        q.put((rank, repr(e)))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def test_two_rank_plan_and_partial_aggregation():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert res == {0: "ok", 1: "ok"}, res


def test_more_ranks_than_clients_gives_empty_shares():
    """K < G: placement leaves some ranks empty; their partial is S = 0, N = 0 and the
    allreduce is unchanged (fl_aggregate handles K_local = 0)."""
    ids, off = fl.fl_place_plan("bu", [0, 1, 2], [5, 9, 1, 4], 4, 8)
    assert list(np.diff(off)) == [1, 1, 1, 0, 0, 0, 0, 0]
