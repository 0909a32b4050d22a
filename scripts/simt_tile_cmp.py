"""θ_new of a small speech round and a small CNN FP32-SIMT (math = 1) round, saved for a
bit-exactness comparison of the SIMT GEMM tile shapes (FL_SIMT_TILE64=1 vs default)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, paper_2306_17453_b200 as fl
out = []
for model, name, math in (("speech", "C4", 0), ("cnn", "C2", 1)):
    wl = synth.preset(name, n_pop=12, n_cohort=12)
    sizes = np.minimum(synth.client_sizes(wl), 90)
    _, x, y = synth.population(wl, sizes)
    ctx = fl.fl_round_init(fl.Config(model=model, batch_size=wl.B, lr=wl.lr, math=math), sizes,
                           torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), synth.init_params(model))
    ctx.fl_round(np.arange(12))
    out.append(ctx.fl_get_global_params())
    ctx.close()
np.save(sys.argv[1], np.concatenate(out))
