"""Is the C2 round host-bound? Host enqueue time of fl_round vs device round time."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, paper_2306_17453_b200 as fl
wl = synth.preset("C2")
sizes = synth.client_sizes(wl)
_, x, y = synth.population(wl, sizes)
ctx = fl.fl_round_init(fl.Config(model="cnn", batch_size=32, lr=wl.lr), sizes, torch.from_numpy(x).cuda(),
                       torch.from_numpy(y).cuda(), synth.init_params("cnn"))
ids = np.arange(len(sizes))
for i in range(3): ctx.fl_round(ids, round_index=i, stats=False)
torch.cuda.synchronize()
enq = []
t0 = time.perf_counter()
for i in range(10):
    a = time.perf_counter(); ctx.fl_round(ids, round_index=10 + i, stats=False); enq.append(time.perf_counter() - a)
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / 10
st = ctx.fl_round(ids, round_index=99)
print(f"host enqueue per round {1e3*np.median(enq):.2f} ms (max {1e3*max(enq):.2f}), wall per round {1e3*wall:.2f} ms, "
      f"device round {st['round_ms']:.2f} ms, place {st['place_ms']:.2f} ms", flush=True)
