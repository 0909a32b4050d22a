"""Heterogeneous-worker emulation on one B200 (§6, Tables 1-4).

Two ranks run as contexts of one process on DISJOINT SM partitions of the same GPU (CUDA green
contexts, include/fl.h sm_count: e.g. 104 + 44 SMs, a ~2.4x speed gap), each driven by its own
host thread, aggregated across ranks over peer memory (FL_AGG_PEER).  The same cohorts are
trained under BU (batch-count load) and under the paper's LB loop (round 0 RR, then one
Eq. 3 fit per GPU from timing records, FL_PLACE_LB_GPU).  Reported per policy:
each rank's training time per round and "timedelta workers" = slowest − fastest rank.
The paper's claim: on heterogeneous hardware LB beats BU because it tells the
workers apart.

    python scripts/hetero_emulation.py [--split 104] [--clients 200] [--rounds 6] [--out f.json]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading

# Two ranks x 9 streams: with the default 8 hardware work queues per process the ranks' streams
# alias onto shared queues and serialise each other (measured: a 104-SM rank 75 -> 190 ms when
# a 44-SM rank trains beside it; 79 ms with 32 queues).  Must be set before CUDA initialises.
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
# Eager module loading: with lazy loading, the first launch of a kernel variant (e.g. a split-K
# shape first met when LB changes a rank's share) loads its module while the peer rank's
# aggregation kernel spins, stalling both ranks for a whole round (seen once in three runs).
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402


class ThreadGroup:
    """allgather across W host threads (one per in-process rank)."""

    def __init__(self, world):
        self.world = world
        self.slots = [None] * world
        self.bar = threading.Barrier(world)

    def allgather(self, rank, arr):
        self.slots[rank] = np.asarray(arr, np.float64).copy()
        self.bar.wait()
        out = np.stack(self.slots)
        self.bar.wait()
        return out


def make_pair(wl, sizes, xd, yd, theta, split):
    import paper_2306_17453_b200 as fl
    ctxs = []
    for r, s in ((0, split), (1, -split)):
        cfg = fl.Config(model=wl.model, batch_size=wl.B, local_epochs=wl.E, lr=wl.lr, shuffle=wl.shuffle,
                        seed=wl.seed, rank=r, world_size=2, sm_count=s, agg_mode="peer")
        ctxs.append(fl.fl_round_init(cfg, sizes, xd, yd, theta))
    blobs = [c.fl_peer_export(0) for c in ctxs]
    for c in ctxs:
        c.fl_peer_connect(blobs)
    return ctxs


def run_policy(policy, ctxs, cohorts, group):
    """Both ranks run every cohort under `policy` ("bu" or "lb"); returns per-round records."""
    from paper_2306_17453_b200.driver import RoundDriver
    out = [[None] * len(cohorts) for _ in ctxs]
    errs = []

    def worker(r):
        try:
            drv = RoundDriver(ctxs[r], policy=policy, allgather=lambda a: group.allgather(r, a))
            for i, c in enumerate(cohorts):
                st = drv.run(c, round_index=i)
                out[r][i] = {"policy": drv.history[-1][0], "train_ms": st["train_ms"],
                             "clients_local": st["clients_local"], "steps_local": st["steps_local"],
                             "round_ms": st["round_ms"], "sm_count": st["sm_count"],
                             "timedelta_ms": st["timedelta_ms"]}
        except Exception as e:  # pragma: no cover - surfaced below
            errs.append(e)
            group.bar.abort()

    th = [threading.Thread(target=worker, args=(r,)) for r in range(len(ctxs))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    if errs:
        raise errs[0]
    rounds = []
    for i in range(len(cohorts)):
        a, b = out[0][i], out[1][i]
        rounds.append({"policy": a["policy"], "train_ms": [a["train_ms"], b["train_ms"]],
                       "clients": [a["clients_local"], b["clients_local"]],
                       "steps": [a["steps_local"], b["steps_local"]],
                       "round_ms_max": max(a["round_ms"], b["round_ms"]), "timedelta_ms": a["timedelta_ms"]})
    return rounds


def experiment(split=104, clients=200, rounds=6, n_pop=10_000, seed=5):
    import torch
    wl = synth.preset("C3", E=1)
    sizes_all = synth.client_sizes(wl)
    rng = np.random.default_rng(seed)
    cohorts_pop = [np.sort(rng.choice(n_pop, size=clients, replace=False)) for _ in range(rounds)]
    ids = np.unique(np.concatenate(cohorts_pop))
    _, x, y = synth.population(wl, sizes_all, clients=ids)
    remap = {int(c): i for i, c in enumerate(ids)}
    sizes = sizes_all[ids]
    cohorts = [np.array([remap[int(c)] for c in co], np.int64) for co in cohorts_pop]
    xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y.astype(np.int32)).cuda()
    theta = synth.init_params("cnn")
    res = {"workload": f"{clients} of {n_pop} CIFAR-shaped clients per round (C3 law, E=1, B=32), "
                       f"{rounds} rounds, two ranks on SM partitions of one B200",
           "split": split}
    for policy in ("bu", "lb"):
        ctxs = make_pair(wl, sizes, xd, yd, theta, split)
        group = ThreadGroup(2)
        run_policy(policy, ctxs, cohorts[:1], group)  # warm-up round (allocations, tensor maps)
        r = run_policy(policy, ctxs, cohorts, group)
        res[policy] = {"sm_count": [c.fl_get_stats()["sm_count"] for c in ctxs], "rounds": r,
                       "timedelta_ms_mean_after_r0": float(np.mean([q["timedelta_ms"] for q in r[1:]])),
                       "round_ms_mean_after_r0": float(np.mean([q["round_ms_max"] for q in r[1:]]))}
        for c in ctxs:
            c.close()
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--split", type=int, default=104)
    ap.add_argument("--clients", type=int, default=200)
    ap.add_argument("--rounds", type=int, default=6)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    res = experiment(a.split, a.clients, a.rounds)
    s = json.dumps(res, indent=1)
    print(json.dumps({p: {k: res[p][k] for k in ("sm_count", "timedelta_ms_mean_after_r0", "round_ms_mean_after_r0")}
                      for p in ("bu", "lb")}))
    if a.out:
        open(a.out, "w").write(s)


if __name__ == "__main__":
    main()
