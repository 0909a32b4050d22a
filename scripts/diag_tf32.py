"""Diagnostic: TF32 (math=0) vs FP32 SIMT (math=1) vs oracle, per tensor, small rounds."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, oracle
import paper_2306_17453_b200 as fl

names = [n for n, _ in synth.param_shapes("cnn")]
sizes_of = [int(np.prod(s)) for _, s in synth.param_shapes("cnn")]
def per_tensor(d):
    out, o = {}, 0
    for n, k in zip(names, sizes_of):
        out[n] = float(np.max(np.abs(d[o:o+k]))); o += k
    return out

def run(sizes, math, lr=0.05, E=1):
    wl = synth.preset("C2", n_pop=len(sizes), n_cohort=len(sizes), lr=lr, E=E)
    _, x, y = synth.population(wl, sizes)
    th = synth.init_params("cnn")
    cfg = fl.Config(model="cnn", batch_size=32, local_epochs=E, lr=lr, math=math)
    ctx = fl.fl_round_init(cfg, sizes, torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), th)
    ctx.fl_place(np.arange(len(sizes))); ctx.fl_train_clients(0)
    tk = [ctx.fl_get_client_params(i) for i in range(len(sizes))]
    out, _ = ctx.fl_aggregate()
    return x, y, th, tk, out

for sizes in [np.array([32]), np.array([64]), np.array([3, 33, 9, 40])]:
    x, y, th, tk0, o0 = run(sizes, 0)
    _, _, _, tk1, o1 = run(sizes, 1)
    ref, _, tkr = oracle.fedavg_round("cnn", th, x, y, sizes, np.arange(len(sizes)), 32, 1, 0.05)
    print("sizes", sizes.tolist())
    print("  tf32 vs oracle", {k: f"{v:.1e}" for k, v in per_tensor(o0 - ref).items()})
    print("  fp32 vs oracle", {k: f"{v:.1e}" for k, v in per_tensor(o1 - ref).items()})
    print("  update magnitude", {k: f"{v:.1e}" for k, v in per_tensor(ref - th).items()})

# C2 full round: tf32 vs fp32 (the fp32 path is oracle-equal to ~1e-6)
wl = synth.preset("C2"); sizes = synth.client_sizes(wl)
x, y, th, tk0, o0 = run(sizes, 0)
_, _, _, tk1, o1 = run(sizes, 1)
d = np.array([np.max(np.abs(a - b)) for a, b in zip(tk0, tk1)])
order = np.argsort(sizes)
print("C2 theta_new tf32-fp32 max", np.max(np.abs(o0 - o1)), per_tensor(o0 - o1))
print("C2 per-client max|tk tf32 - fp32| by size:", [(int(sizes[i]), f"{d[i]:.1e}") for i in order[::10]])
