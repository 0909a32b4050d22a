"""Host issue cost of one C2 round with the GPU stalled behind a long kernel (queue never drains)."""
import os, sys, time
os.environ["FL_HOSTPROF"] = "1"
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
print("--- GPU free-running", flush=True)
for i in range(2): ctx.fl_round(ids, round_index=5 + i, stats=False)
torch.cuda.synchronize()
print("--- GPU stalled by a long sleep on the ctx stream", flush=True)
s = torch.cuda.ExternalStream(ctx.stream)
with torch.cuda.stream(s):
    torch.cuda._sleep(400_000_000)
ctx.fl_round(ids, round_index=9, stats=False)
torch.cuda.synchronize()
