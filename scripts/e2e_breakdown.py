"""Host wall-clock breakdown of the e2e C2 round (public API, host population)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, paper_2306_17453_b200 as fl
wl = synth.preset("C2")
sizes = synth.client_sizes(wl)
_, x, y = synth.population(wl, sizes)
ctx = fl.fl_round_init(fl.Config(model="cnn", batch_size=32, lr=wl.lr), sizes, x, y, synth.init_params("cnn"),
                       on_device=False)
ids = np.arange(len(sizes))
T = []
for r in range(8):
    t0 = time.perf_counter(); ctx.fl_place(ids)
    t1 = time.perf_counter(); ctx.fl_train_clients(r)
    t2 = time.perf_counter(); ctx.fl_aggregate(want_params=True)
    t3 = time.perf_counter()
    st = ctx.fl_get_stats()
    T.append((t1 - t0, t2 - t1, t3 - t2, t3 - t0, st["round_ms"] / 1e3, st["stage_ms"] / 1e3, st["train_ms"] / 1e3))
for row in T[3:]:
    print("place %.2f  train(host) %.2f  aggregate+sync %.2f  total %.2f | device round %.2f stage %.2f train %.2f ms" %
          tuple(1e3 * v for v in row))
