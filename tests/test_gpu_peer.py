"""GPU tests of the SM-partitioned ranks (green contexts, include/fl.h sm_count) and of the
cross-rank aggregation over peer memory (FL_AGG_PEER, FL_AGG_UNAGGREGATED).

Two ranks share the one B200 of the test box as contexts of one process on disjoint SM
partitions, so the whole multi-rank protocol (plan on every rank, local SGD of each rank's
share, partial fp64 aggregation, reduce-scatter + finalize + all-gather over peer memory, or
every client model shipped to the server rank) runs for real.  Bars as in test_gpu_parity:
θ_new within 1e-3 of the oracle's round (A21), aggregation alone within 1e-6 (R9/A20), and
both ranks hold the same θ_new bit for bit.
"""
import numpy as np
import pytest

import oracle
import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2306_17453_b200 as fl  # noqa: E402

TOL_ROUND = 1e-3
TOL_AGG = 1e-6


def agg_err(gpu, theta_k, n):
    o, _ = oracle.fedavg(theta_k.astype(np.float64), n)
    w = np.asarray(n, np.float64) / np.sum(n)
    s = np.abs(theta_k.astype(np.float64)).T @ w
    return float(np.max(np.abs(gpu.astype(np.float64) - o) / np.maximum(s, 1e-30)))


def small_cnn(n_pop=12, seed=3):
    wl = synth.preset("C2", n_pop=n_pop, n_cohort=n_pop)
    rng = np.random.default_rng(seed)
    sizes = rng.integers(5, 100, size=n_pop).astype(np.int64)
    _, x, y = synth.population(wl, sizes)
    return wl, sizes, x, y, synth.init_params("cnn")


def make(wl, sizes, xd, yd, theta, **kw):
    cfg = fl.Config(model=wl.model, batch_size=wl.B, local_epochs=wl.E, lr=wl.lr, shuffle=wl.shuffle, seed=wl.seed,
                    **kw)
    return fl.fl_round_init(cfg, sizes, xd, yd, theta)


def pair(wl, sizes, x, y, theta, mode, split=74, max_clients=0):
    """Two ranks of one process on disjoint SM partitions of device 0, peer-connected."""
    xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y.astype(np.int32)).cuda()
    r0 = make(wl, sizes, xd, yd, theta, rank=0, world_size=2, sm_count=split, agg_mode=mode)
    r1 = make(wl, sizes, xd, yd, theta, rank=1, world_size=2, sm_count=-split, agg_mode=mode)
    blobs = [r0.fl_peer_export(max_clients), r1.fl_peer_export(0)]
    r0.fl_peer_connect(blobs)
    r1.fl_peer_connect(blobs)
    return r0, r1, (xd, yd)


def test_green_partition_round_matches_oracle():
    """A rank on a 48-SM partition: its streams run there, persistent grids are sized to it,
    and the round still matches the oracle."""
    wl, sizes, x, y, theta = small_cnn()
    xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y.astype(np.int32)).cuda()
    ctx = make(wl, sizes, xd, yd, theta, sm_count=48)
    st = ctx.fl_round(np.arange(len(sizes)))
    assert 48 <= st["sm_count"] < 148
    ref, N, _ = oracle.fedavg_round("cnn", theta, x, y, sizes, np.arange(len(sizes)), wl.B, wl.E, wl.lr)
    assert float(np.max(np.abs(ctx.fl_get_global_params() - ref))) <= TOL_ROUND
    ctx.close()
    rem = make(wl, sizes, xd, yd, theta, sm_count=-48)
    st = rem.fl_round(np.arange(len(sizes)))
    assert 0 < st["sm_count"] <= 100
    rem.close()


@pytest.mark.parametrize("mode", ["peer", "unaggregated"])
def test_two_ranks_peer_aggregation_vs_oracle(mode):
    wl, sizes, x, y, theta = small_cnn()
    K = len(sizes)
    r0, r1, keep = pair(wl, sizes, x, y, theta, mode, max_clients=K)
    rng = np.random.default_rng(7)
    cohorts = [rng.choice(K, size=k, replace=False) for k in (12, 5, 9)]
    th = theta.astype(np.float32)
    for rnd, c in enumerate(cohorts):
        # aggregation alone: θ_k read back from the rank that trained each client
        for r in (r0, r1):
            r.fl_place(c)
            r.fl_train_clients(rnd)
        ids0, _, _ = r0.fl_get_local_plan()
        ids1, _, _ = r1.fl_get_local_plan()
        assert len(ids0) + len(ids1) == len(c) and len(ids0) > 0 and len(ids1) > 0
        tk = np.stack([r0.fl_get_client_params(k) for k in ids0] + [r1.fl_get_client_params(k) for k in ids1])
        n = sizes[np.concatenate([ids0, ids1])]
        out0, N0 = r0.fl_aggregate(want_params=False)
        out1, N1 = r1.fl_aggregate(want_params=False)
        a, b = r0.fl_get_global_params(), r1.fl_get_global_params()
        assert np.array_equal(a, b), float(np.max(np.abs(a - b)))
        assert N0 == N1 == sizes[c].sum()
        assert agg_err(a, tk, n) <= TOL_AGG
        ref, _, _ = oracle.fedavg_round("cnn", th, x, y, sizes, c, wl.B, wl.E, wl.lr, rnd=rnd)
        assert float(np.max(np.abs(a - ref))) <= TOL_ROUND
        th = a
        s0, s1 = r0.fl_get_stats(), r1.fl_get_stats()
        P = fl.fl_n_params("cnn")
        if mode == "unaggregated":  # every client model of rank 1 crosses to the server
            assert s1["xfer_bytes"] >= 4 * P * len(ids1) and s0["xfer_bytes"] >= 4 * P
        else:  # half of S pulled (8 B) and half of θ_new pushed (4 B) per rank
            assert 5.5 * P <= s0["xfer_bytes"] <= 6.5 * P and 5.5 * P <= s1["xfer_bytes"] <= 6.5 * P
    r0.close()
    r1.close()


def test_peer_queued_rounds_match_single_gpu():
    """fl_round with stats=False on both ranks, several rounds queued with no host sync: the
    sequence-numbered signals keep the rounds apart; θ_new equals the oracle's rounds."""
    wl, sizes, x, y, theta = small_cnn(n_pop=10, seed=9)
    r0, r1, keep = pair(wl, sizes, x, y, theta, "peer", split=100)
    rng = np.random.default_rng(3)
    cohorts = [rng.choice(10, size=k, replace=False) for k in (10, 4, 7, 3)]
    for rnd, c in enumerate(cohorts):
        r0.fl_round(c, round_index=rnd, stats=False)
        r1.fl_round(c, round_index=rnd, stats=False)
    a, b = r0.fl_get_global_params(), r1.fl_get_global_params()
    assert np.array_equal(a, b)
    th = theta.astype(np.float32)
    for rnd, c in enumerate(cohorts):
        th, _, _ = oracle.fedavg_round("cnn", th.astype(np.float32), x, y, sizes, c, wl.B, wl.E, wl.lr, rnd=rnd)
    assert float(np.max(np.abs(a - th))) <= TOL_ROUND
    r0.close()
    r1.close()


def test_peer_world1_equals_fused_path_bitwise():
    """world 1 through the peer kernel: the same fp64 arithmetic in the same client order as
    the fused single-GPU accumulate+finalize, so θ_new is bit-identical."""
    wl, sizes, x, y, theta = small_cnn(n_pop=8, seed=4)
    xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y.astype(np.int32)).cuda()
    p = make(wl, sizes, xd, yd, theta, agg_mode="peer")
    p.fl_peer_connect([p.fl_peer_export(0)])
    f = make(wl, sizes, xd, yd, theta)
    for rnd in range(2):
        p.fl_round(np.arange(8), round_index=rnd, stats=False)
        f.fl_round(np.arange(8), round_index=rnd, stats=False)
    assert np.array_equal(p.fl_get_global_params(), f.fl_get_global_params())
    p.close()
    f.close()


def test_shared_device_without_partitions_rejected():
    wl, sizes, x, y, theta = small_cnn(n_pop=4)
    xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y.astype(np.int32)).cuda()
    r0 = make(wl, sizes, xd, yd, theta, rank=0, world_size=2, agg_mode="peer")
    r1 = make(wl, sizes, xd, yd, theta, rank=1, world_size=2, agg_mode="peer")
    blobs = [r0.fl_peer_export(0), r1.fl_peer_export(0)]
    with pytest.raises(fl.FLError) as e:
        r0.fl_peer_connect(blobs)
    assert e.value.status == fl.FL_ERR_INVALID
    with pytest.raises(fl.FLError):
        r0.fl_round(np.arange(4))  # world 2 peer mode without a connection: FL_ERR_STATE
    r0.close()
    r1.close()


def test_heterogeneous_ranks_lb_beats_bu(tmp_path):
    """SURVEY §8 f4 / P:427-430: two ranks on 104- and 44-SM partitions (a ~2.1x speed gap
    measured alone).  BU balances batch counts, so the slow rank finishes long after the fast
    one; the LB loop (RR bootstrap, per-GPU Eq. 3 fits from timing records) gives the fast
    rank more work and cuts "timedelta workers".  Run in a subprocess: the two
    ranks' 18 streams need CUDA_DEVICE_MAX_CONNECTIONS=32 and eager module loading, set before CUDA
    initialises."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, CUDA_DEVICE_MAX_CONNECTIONS="32", CUDA_MODULE_LOADING="EAGER")

    def slow_rank_ms_per_step(res):
        return [r["train_ms"][1] / max(r["steps"][1], 1) for p in ("bu", "lb") for r in res[p]["rounds"]]

    # Emulation validity: the partitions' speeds must stay put.  Two ranks in one process share
    # HBM, L2 and the hardware work queues; in some runs (seen with the round-1 kernels too) the
    # 44-SM rank's streams get serialised behind the other rank's for the whole experiment, its
    # time per SGD step inflating 2-5x for the same work, which no placement rule can fix.  Such
    # a run is detected from the slow rank's ms per step (> 1.6x its minimum) and re-run once.
    for attempt in range(2):
        out = tmp_path / f"hetero{attempt}.json"
        subprocess.run([sys.executable, os.path.join(root, "scripts", "hetero_emulation.py"), "--clients", "1000",
                        "--rounds", "6", "--out", str(out)], check=True, env=env, timeout=600)
        res = json.load(open(out))
        mps = slow_rank_ms_per_step(res)
        print(f"attempt {attempt}: slow-rank ms/step {min(mps):.4f}..{max(mps):.4f}")
        if max(mps) <= 1.6 * min(mps):
            break
    bu, lb = res["bu"], res["lb"]
    assert bu["sm_count"][0] > 1.5 * bu["sm_count"][1]
    print(f"timedelta BU {bu['timedelta_ms_mean_after_r0']:.2f} ms, LB {lb['timedelta_ms_mean_after_r0']:.2f} ms")
    # measured over 6 runs of 1,000 clients: BU 88 ms, LB 39-66 ms (the LB placements vary with the
    # timing records each round's fits see)
    assert lb["timedelta_ms_mean_after_r0"] < 0.85 * bu["timedelta_ms_mean_after_r0"]
    assert lb["round_ms_mean_after_r0"] < bu["round_ms_mean_after_r0"]
    # LB moves work to the faster partition: more SGD steps on rank 0 than BU gives it
    assert np.mean([r["steps"][0] for r in lb["rounds"][1:]]) > np.mean([r["steps"][0] for r in bu["rounds"][1:]])
