"""A few char-LSTM rounds of A clients x 4 steps (for ncu launch lists). usage: lstm_one.py [A]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, paper_2306_17453_b200 as fl
A = int(sys.argv[1]) if len(sys.argv) > 1 else 1
sizes = np.full(A, 16, dtype=np.int64)
wl = synth.preset("C5", n_pop=A, n_cohort=A)
_, x, y = synth.population(wl, sizes)
cfg = fl.Config(model="lstm", batch_size=4, local_epochs=1, lr=wl.lr)
c = fl.fl_round_init(cfg, sizes, torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), synth.init_params("lstm"))
for i in range(2):
    print(c.fl_round(np.arange(A), round_index=i)["round_ms"], flush=True)
