"""One char-LSTM round of a C5-law cohort (for ncu launch lists): usage lstm_round.py K rounds"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, paper_2306_17453_b200 as fl
K, rounds = (int(a) for a in (sys.argv[1:] + ["64", "2"])[:2])
wl = synth.preset("C5", n_pop=K, n_cohort=K)
sizes = synth.client_sizes(wl)
_, x, y = synth.population(wl, sizes)
ctx = fl.fl_round_init(fl.Config(model="lstm", batch_size=wl.B, lr=wl.lr), sizes, torch.from_numpy(x).cuda(),
                       torch.from_numpy(y).cuda(), synth.init_params("lstm"))
for r in range(rounds):
    print(ctx.fl_round(np.arange(K), round_index=r)["round_ms"], flush=True)
