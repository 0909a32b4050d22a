import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import synth, paper_2306_17453_b200 as fl
wl = synth.preset("C5", n_pop=24, n_cohort=24)
sizes = synth.client_sizes(wl); sizes = np.minimum(sizes, 40)
_, x, y = synth.population(wl, sizes)
ctx = fl.fl_round_init(fl.Config(model="lstm", batch_size=4, lr=wl.lr), sizes, torch.from_numpy(x).cuda(),
                       torch.from_numpy(y).cuda(), synth.init_params("lstm"))
ctx.fl_round(np.arange(24))
np.save(sys.argv[1], ctx.fl_get_global_params())
