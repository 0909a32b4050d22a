"""One client of 2000 samples, one round (for ncu launch lists of the critical path)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, paper_2306_17453_b200 as fl
sizes = np.array([int(sys.argv[1]) if len(sys.argv) > 1 else 2000])
wl = synth.preset("C2", n_pop=1, n_cohort=1)
_, x, y = synth.population(wl, sizes)
ctx = fl.fl_round_init(fl.Config(model="cnn", batch_size=32, lr=wl.lr), sizes, torch.from_numpy(x).cuda(),
                       torch.from_numpy(y).cuda(), synth.init_params("cnn"))
for i in range(2):
    print(ctx.fl_round(np.arange(1), round_index=i)["round_ms"])
