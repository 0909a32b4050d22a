"""Debug: unaggregated / peer aggregation with logreg (tiny), world 1 or 2 in-process ranks."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, paper_2306_17453_b200 as fl
mode, world = sys.argv[1], int(sys.argv[2])
wl = synth.preset("C1", n_pop=12, n_cohort=12)
sizes = synth.client_sizes(wl)
_, x, y = synth.population(wl, sizes)
theta = synth.init_params("logreg")
xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y.astype(np.int32)).cuda()
rs = []
for r in range(world):
    s = 0 if world == 1 else (74 if r == 0 else -74)
    cfg = fl.Config(model="logreg", batch_size=wl.B, lr=wl.lr, rank=r, world_size=world, sm_count=s, agg_mode=mode)
    rs.append(fl.fl_round_init(cfg, sizes, xd, yd, theta))
blobs = [c.fl_peer_export(12 if i == 0 else 0) for i, c in enumerate(rs)]
for c in rs: c.fl_peer_connect(blobs)
for rnd in range(2):
    for c in rs:
        c.fl_place(np.arange(12)); c.fl_train_clients(rnd)
    for c in rs:
        c.fl_aggregate(want_params=False)
    torch.cuda.synchronize()
    print(mode, world, "round", rnd, "ok", [c.fl_get_stats()["xfer_bytes"] for c in rs], flush=True)
