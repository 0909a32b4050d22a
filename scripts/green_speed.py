"""Training speed of SM partitions (green contexts), alone and concurrently: two world-1 ctxs
on disjoint partitions of one B200 each training half of a C3-law cohort."""
import os, sys, threading, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, paper_2306_17453_b200 as fl
split = int(sys.argv[1]) if len(sys.argv) > 1 else 104
clients = int(sys.argv[2]) if len(sys.argv) > 2 else 500
wl = synth.preset("C3", E=1)
sizes_all = synth.client_sizes(wl)
ids = np.sort(np.random.default_rng(5).choice(10000, size=clients, replace=False))
_, x, y = synth.population(wl, sizes_all, clients=ids)
sizes = sizes_all[ids]
xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y.astype(np.int32)).cuda()
theta = synth.init_params("cnn")
def mk(s):
    return fl.fl_round_init(fl.Config(model="cnn", batch_size=32, lr=wl.lr, sm_count=s), sizes, xd, yd, theta)
res = {}
for s in (0, split, -split):
    c = mk(s)
    c.fl_round(np.arange(clients))
    st = [c.fl_round(np.arange(clients), round_index=i) for i in range(3)]
    res[f"alone sm_count={s}"] = {"sms": st[0]["sm_count"], "train_ms": [q["train_ms"] for q in st]}
    c.close()
cs = [mk(split), mk(-split)]
for c in cs: c.fl_round(np.arange(clients))
out = [None, None]
def w(i):
    out[i] = [cs[i].fl_round(np.arange(clients), round_index=r)["train_ms"] for r in range(3)]
th = [threading.Thread(target=w, args=(i,)) for i in range(2)]
[t.start() for t in th]; [t.join() for t in th]
res["concurrent"] = {"train_ms_rank0": out[0], "train_ms_rank1": out[1]}
print(json.dumps(res, indent=1))
