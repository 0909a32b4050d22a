"""Per-client completion times of one C2 round (LB timing records): is the round bound by the
bulk groups' throughput or by the largest clients' step latency?"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, paper_2306_17453_b200 as fl
wl = synth.preset("C2")
sizes = synth.client_sizes(wl)
_, x, y = synth.population(wl, sizes)
ctx = fl.fl_round_init(fl.Config(model="cnn", batch_size=32, lr=wl.lr), sizes, torch.from_numpy(x).cuda(),
                       torch.from_numpy(y).cuda(), synth.init_params("cnn"))
ids = np.arange(len(sizes))
for i in range(3):
    ctx.fl_round(ids, round_index=i, stats=False)
ctx.fl_set_timing_records(True)
st = ctx.fl_round(ids, round_index=3)
cid, m, t = ctx.fl_get_client_times()
o = np.argsort(-t)
print("round_ms %.3f train_ms %.3f stage_ms %.3f" % (st["round_ms"], st["train_ms"], st["stage_ms"]))
for j in o[:12]:
    print("client %3d m=%3d done at %.3f ms" % (cid[j], m[j], t[j]))
print("m quantiles", np.percentile(m, [50, 90, 100]), "t quantiles", np.percentile(t, [50, 90, 100]))
# one client alone
for mm in sorted(set(m.tolist()))[-3:]:
    j = int(np.where(m == mm)[0][0])
    st1 = ctx.fl_round(np.array([cid[j]]), round_index=9)
    print("alone: client m=%d round %.3f ms (%.1f us/step)" % (mm, st1["round_ms"], st1["round_ms"] * 1e3 / mm))
