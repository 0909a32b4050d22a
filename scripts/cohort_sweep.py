#!/usr/bin/env python
"""Clients-per-round sweep (Table 3).

10,000-client CIFAR-shaped population (C3's size law), cohorts of 100 / 200 / 400 /
625 / 1,000 clients drawn uniformly without replacement per round (reading A19),
McMahan CNN, B = 32, E = 2 (C3), one B200.  Each cohort size runs W warm-up rounds
and R timed rounds through RoundDriver (policy BU, or the LB loop with --policy lb);
every round draws a fresh cohort.  Device time per round from the library's own
events (fl_round_stats.round_ms); throughput = clients / round time.

    python scripts/cohort_sweep.py [--rounds 5] [--warmup 2] [--policy bu|lb] [--out gpurun_out/cohort_sweep.json]
"""
import argparse
import json
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rounds", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--policy", default="bu")
    ap.add_argument("--sizes", default="100,200,400,625,1000")
    ap.add_argument("--E", type=int, default=2)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "cohort_sweep.json"))
    args = ap.parse_args()
    import torch
    import paper_2306_17453_b200 as fl
    from paper_2306_17453_b200.driver import RoundDriver, sample_cohort

    wl = synth.preset("C3", E=args.E)
    sizes = synth.client_sizes(wl)
    x, y = synth.population_torch(wl, sizes, "cuda")
    theta = synth.init_params("cnn")
    cfg = fl.Config(model="cnn", batch_size=wl.B, local_epochs=wl.E, lr=wl.lr, seed=wl.seed)
    ctx = fl.fl_round_init(cfg, sizes, x, y, theta)
    rows = []
    rnd = 0
    for K in [int(v) for v in args.sizes.split(",")]:
        drv = RoundDriver(ctx, policy=args.policy)
        ms = []
        for i in range(args.warmup + args.rounds):
            st = drv.run(sample_cohort(wl.n_pop, K, wl.seed, rnd), rnd)
            rnd += 1
            if i >= args.warmup:
                ms.append(st["round_ms"])
        med = statistics.median(ms)
        row = {"clients_per_round": K, "population": wl.n_pop, "E": wl.E, "B": wl.B, "policy": args.policy,
               "rounds": args.rounds, "round_ms_median": med, "round_ms_min": min(ms), "round_ms_max": max(ms),
               "client_updates_per_s": K / (med * 1e-3)}
        rows.append(row)
        print(json.dumps(row), flush=True)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump({"workload": "C3 population (10,000 CIFAR-shaped clients), McMahan CNN, 1 B200",
                   "gpu": torch.cuda.get_device_name(0), "rows": rows}, f, indent=1)
    ctx.close()


if __name__ == "__main__":
    main()
