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


# ------------------------------------------------------------------ LB loop across ranks (f1, f4)
class _FakeCtx:
    """Stands in for a rank's fl_ctx on CPU: placement through the library's host planner,
    training time from a per-rank cost model t = speed · m (a heterogeneous pair of GPUs,
    PAPER.md L427-430), completion records as fl_get_client_times returns them."""

    def __init__(self, rank, world, sizes, B, speed):
        self.cfg = type("C", (), {"world_size": world, "rank": rank})()
        self.rank, self.world, self.sizes, self.B, self.speed = rank, world, sizes, B, speed
        self.seen = []

    def fl_set_timing_records(self, on=True):
        pass

    def fl_round(self, cohort, policy="bu", lb_coef=None, round_index=0):
        ids, off = fl.fl_place_plan(policy, cohort, self.sizes, self.B, self.world, lb_coef)
        self.seen.append((policy, None if lb_coef is None else np.array(lb_coef)))
        self.local = ids[off[self.rank]:off[self.rank + 1]]
        m = (self.sizes[self.local] + self.B - 1) // self.B
        self.t = self.speed * m.astype(np.float64) + 0.5  # per-client job time of this GPU (L378)
        return {"train_ms": float(self.speed * m.sum()), "clients_total": len(cohort)}

    def fl_get_client_times(self):
        m = (self.sizes[self.local] + self.B - 1) // self.B
        return self.local, m, self.t


def _lb_worker(rank, world, port, q):
    try:
        from paper_2306_17453_b200.driver import RoundDriver, sample_cohort
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)

        def allgather(v):
            out = [None] * world
            dist.all_gather_object(out, np.asarray(v, np.float64).tolist())
            return np.array(out)

        wl = synth.preset("C3", n_pop=400, n_cohort=120)
        sizes = synth.client_sizes(wl)
        ctx = _FakeCtx(rank, world, sizes, wl.B, speed=1.0 if rank == 0 else 3.0)
        drv = RoundDriver(ctx, policy="lb", allgather=allgather)
        loads = []
        for r in range(3):
            st = drv.run(sample_cohort(400, 120, wl.seed, r), r)
            loads.append(allgather([st["train_ms"], 0, 0, 0])[:, 0].tolist())
        q.put((rank, [p for p, _ in ctx.seen], drv.coef.tolist(), loads, st["timedelta_ms"]))
    except Exception as e:  # pragma: no cover
        q.put((rank, "error", repr(e), None, None))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def test_lb_loop_two_ranks_heterogeneous():
    """RR bootstrap (L375), then every rank fits its own records (L378) and all ranks place
    with the same gathered per-GPU fits (FL_PLACE_LB_GPU): the 3x slower rank gets ~1/3 of
    the batches and the timedelta (L412) shrinks from RR's."""
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_lb_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=240) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
    for rank, pols, coef, loads, td in res:
        assert pols != "error", coef
        assert pols == ["rr", "lb_gpu", "lb_gpu"]
        # both ranks hold the same gathered fits; rank 1's slope is 3x rank 0's
        assert np.allclose(coef, res[0][2])
        assert coef[1][0] == pytest.approx(3 * coef[0][0], rel=1e-6)
    loads = res[0][3]
    rr_gap = abs(loads[0][0] - loads[0][1]) / max(loads[0])
    lb_gap = abs(loads[2][0] - loads[2][1]) / max(loads[2])
    assert lb_gap < 0.1 < rr_gap, (loads, rr_gap, lb_gap)
    assert res[0][4] == pytest.approx(abs(loads[2][0] - loads[2][1]))


# ------------------------------------------------------------------ peer-memory blob exchange (f3)
class _BlobCtx:
    """Stands in for a rank's fl_ctx: fl_peer_export returns a rank-stamped blob (the real one
    carries CUDA IPC handles), fl_peer_connect records what it was given."""

    def __init__(self, rank):
        self.cfg = type("C", (), {"rank": rank})()
        self.got = None
        self.max_clients = None

    def fl_peer_export(self, max_clients=0):
        self.max_clients = max_clients
        return bytes([self.cfg.rank]) * fl.PEER_BLOB_BYTES

    def fl_peer_connect(self, blobs):
        self.got = blobs


def _blob_worker(rank, world, port, q):
    try:
        import bench
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        ctx = _BlobCtx(rank)
        bench.peer_connect(ctx, world, max_clients=1000)
        q.put((rank, [b[0] for b in ctx.got], [len(b) for b in ctx.got], ctx.max_clients))
    except Exception as e:  # pragma: no cover
        q.put((rank, "error", repr(e), None))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def test_peer_blob_exchange_two_ranks():
    """bench.peer_connect all-gathers every rank's blob in rank order; only the server (rank 0)
    asks for a receive buffer (the unaggregated ablation ships client models to it)."""
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_blob_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = sorted(q.get(timeout=240) for _ in range(world))
    for p in ps:
        p.join(timeout=60)
    for rank, order, lens, maxc in res:
        assert order == [0, 1], (rank, order)
        assert lens == [fl.PEER_BLOB_BYTES] * world
        assert maxc == (1000 if rank == 0 else 0)
