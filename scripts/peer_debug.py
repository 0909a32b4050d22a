"""Debug: one unaggregated / peer round on two in-process ranks, dumping signal words."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, paper_2306_17453_b200 as fl
mode = sys.argv[1] if len(sys.argv) > 1 else "unaggregated"
wl = synth.preset("C2", n_pop=12, n_cohort=12)
sizes = np.random.default_rng(3).integers(5, 100, size=12).astype(np.int64)
_, x, y = synth.population(wl, sizes)
theta = synth.init_params("cnn")
xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y.astype(np.int32)).cuda()
rs = []
for r, s in ((0, 74), (1, -74)):
    cfg = fl.Config(model="cnn", batch_size=32, lr=wl.lr, rank=r, world_size=2, sm_count=s, agg_mode=mode)
    rs.append(fl.fl_round_init(cfg, sizes, xd, yd, theta))
blobs = [rs[0].fl_peer_export(12), rs[1].fl_peer_export(0)]
for c in rs: c.fl_peer_connect(blobs)
T = (2157312 + 8191) // 8192
for rnd in range(3):
    for c in rs:
        c.fl_place(np.arange(12)); c.fl_train_clients(rnd)
    torch.cuda.synchronize()
    print("trained", rnd, flush=True)
    for c in rs:
        c.fl_aggregate(want_params=False)
    for it in range(20):
        time.sleep(0.25)
        for i, c in enumerate(rs):
            s = c.fl_debug_read("sig", (9 * T,), np.uint64)
            print(rnd, it, "rank", i, "ready0[:4]", s[:4], "ready1[:2]", s[T:T + 2], "done[:2]", s[2 * T:2 * T + 2], flush=True)
    print("params equal", np.array_equal(rs[0].fl_get_global_params(), rs[1].fl_get_global_params()), flush=True)
