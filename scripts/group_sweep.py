"""C2 round time for one (FL_SOLO, FL_GROUPS) setting (env), median of 10 rounds."""
import os, sys
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
ms = [ctx.fl_round(ids, round_index=3 + i)["round_ms"] for i in range(10)]
print(f"solo={os.environ.get('FL_SOLO','-')} groups={os.environ.get('FL_GROUPS','-')} round={np.median(ms):.2f} ms "
      f"min={min(ms):.2f}", flush=True)
