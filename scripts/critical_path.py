"""Critical-path study: C2 round vs rounds with the same total samples but no size tail."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, paper_2306_17453_b200 as fl

def run(sizes, steps=5, warm=3, label=""):
    wl = synth.preset("C2", n_pop=len(sizes), n_cohort=len(sizes))
    _, x, y = synth.population(wl, sizes)
    ctx = fl.fl_round_init(fl.Config(model="cnn", batch_size=32, lr=wl.lr), sizes, torch.from_numpy(x).cuda(),
                           torch.from_numpy(y).cuda(), synth.init_params("cnn"))
    for i in range(warm): ctx.fl_round(np.arange(len(sizes)), round_index=i, stats=False)
    ms = [ctx.fl_round(np.arange(len(sizes)), round_index=warm + i)["round_ms"] for i in range(steps)]
    ctx.fl_set_profiling(True); ctx.fl_round(np.arange(len(sizes)), round_index=99)
    ks = ctx.fl_get_kernel_stats()
    print(f"{label:28s} clients={len(sizes):4d} samples={int(sizes.sum()):6d} waves={int(np.ceil(sizes.max()/32)):3d} "
          f"round={np.median(ms):7.2f} ms  sum(kernels)={sum(v['ms'] for v in ks.values()):7.2f} ms", flush=True)

c2 = synth.client_sizes(synth.preset("C2"))
if len(sys.argv) > 1: run = lambda *a, **k: None
run(c2, label="C2 (log-normal)")
run(np.full(100, int(c2.mean())), label="C2 equal sizes")
run(np.array([2000]), label="largest client alone")
run(np.array([int(c2.mean())] * 1), label="one mean client")
run(np.sort(c2)[:-1], label="C2 without largest")

def table(sizes, label):
    wl = synth.preset("C2", n_pop=len(sizes), n_cohort=len(sizes))
    _, x, y = synth.population(wl, sizes)
    ctx = fl.fl_round_init(fl.Config(model="cnn", batch_size=32, lr=wl.lr), sizes, torch.from_numpy(x).cuda(),
                           torch.from_numpy(y).cuda(), synth.init_params("cnn"))
    for i in range(3): ctx.fl_round(np.arange(len(sizes)), round_index=i, stats=False)
    ctx.fl_set_profiling(True); st = ctx.fl_round(np.arange(len(sizes)), round_index=99)
    ks = ctx.fl_get_kernel_stats()
    print(f"--- {label}: round {st['round_ms']:.2f} ms")
    for k, v in sorted(ks.items(), key=lambda kv: -kv[1]["ms"]):
        per = v["ms"] / v["launches"] * 1e3
        extra = f"{v['flops']/v['ms']/1e9:8.1f} TF/s" if v["flops"] else f"{v['bytes']/v['ms']/1e6:8.1f} GB/s"
        print(f"   {k:22s} {v['ms']:7.3f} ms  {v['launches']:3d} x {per:7.1f} us  {extra}")

if len(sys.argv) > 1:
    table(np.full(100, int(c2.mean())), "C2 equal sizes")
    table(np.array([2000]), "largest client alone")
