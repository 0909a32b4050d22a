"""Rounds of A equal clients (|b| = 32, `steps` steps each) in one group, for ncu captures.
usage: wave_once.py A steps rounds"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("FL_SOLO", "0")
os.environ.setdefault("FL_GROUPS", "1")
import numpy as np, torch
import synth, paper_2306_17453_b200 as fl
A, steps, rounds = (int(a) for a in (sys.argv[1:] + ["100", "2", "2"])[:3])
sizes = np.full(A, 32 * steps)
wl = synth.preset("C2", n_pop=A, n_cohort=A)
_, x, y = synth.population(wl, sizes)
ctx = fl.fl_round_init(fl.Config(model="cnn", batch_size=32, lr=wl.lr), sizes, torch.from_numpy(x).cuda(),
                       torch.from_numpy(y).cuda(), synth.init_params("cnn"))
for i in range(rounds):
    print(ctx.fl_round(np.arange(A), round_index=i)["round_ms"], flush=True)
