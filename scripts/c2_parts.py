"""C2 round decomposed: the whole cohort vs its 4 longest clients alone vs the rest alone."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, paper_2306_17453_b200 as fl

def run(sizes, label):
    wl = synth.preset("C2", n_pop=len(sizes), n_cohort=len(sizes))
    _, x, y = synth.population(wl, sizes)
    ctx = fl.fl_round_init(fl.Config(model="cnn", batch_size=32, lr=wl.lr), sizes, torch.from_numpy(x).cuda(),
                           torch.from_numpy(y).cuda(), synth.init_params("cnn"))
    ids = np.arange(len(sizes))
    for i in range(3): ctx.fl_round(ids, round_index=i, stats=False)
    ms = [ctx.fl_round(ids, round_index=3 + i)["round_ms"] for i in range(5)]
    st = ctx.fl_get_stats()
    print(f"{label:34s} clients={len(sizes):3d} steps={int(np.ceil(sizes / 32).sum()):4d} round={np.median(ms):6.2f} ms "
          f"waves={st['waves']}", flush=True)
    ctx.close()

c2 = np.sort(synth.client_sizes(synth.preset("C2")))[::-1]
run(c2, "C2")
run(c2[:4], "4 longest")
run(c2[:1], "longest")
run(c2[4:], "C2 minus 4 longest")
run(c2[1:], "C2 minus longest")
