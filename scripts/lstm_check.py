"""char-LSTM (C5) on the GPU: parity magnitudes vs the oracle, per-wave times, one C5 round."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, oracle, paper_2306_17453_b200 as fl

def ctx_for(wl, sizes):
    _, x, y = synth.population(wl, sizes)
    th = synth.init_params("lstm")
    cfg = fl.Config(model="lstm", batch_size=4, local_epochs=wl.E, lr=wl.lr, shuffle=wl.shuffle, seed=wl.seed)
    return fl.fl_round_init(cfg, sizes, torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), th), x, y, th

sizes = np.array([1, 3, 4, 5, 9, 16], dtype=np.int64)
wl = synth.preset("C5", n_pop=len(sizes), n_cohort=len(sizes), E=2, shuffle=1)
ctx, x, y, th = ctx_for(wl, sizes)
ids = np.arange(len(sizes))
ctx.fl_place(ids); ctx.fl_train_clients(0)
tk = [ctx.fl_get_client_params(i) for i in ids]
out, N = ctx.fl_aggregate()
ref, Nref, tko = oracle.fedavg_round("lstm", th, x, y, sizes, ids, 4, wl.E, wl.lr, wl.shuffle, wl.seed, 0, 0)
print("E=2 shuffled: per-client max|Δθ_k| =", [f"{np.max(np.abs(tk[i] - tko[i])):.2e}" for i in ids],
      " θ_new max|Δ| =", f"{np.max(np.abs(out - ref)):.2e}", " max|θ_new-θ_g| =", f"{np.max(np.abs(out - th)):.2e}", flush=True)
for A in [1, 8, 32, 148]:
    s = np.full(A, 4 * 4, dtype=np.int64)  # 4 steps each
    w = synth.preset("C5", n_pop=A, n_cohort=A)
    c, *_ = ctx_for(w, s)
    for i in range(2): c.fl_round(np.arange(A), round_index=i, stats=False)
    ms = np.median([c.fl_round(np.arange(A), round_index=3 + i)["round_ms"] for i in range(3)])
    print(f"A={A:4d}: {ms / 4:.3f} ms per wave, {ms / 4 / A * 1e3:.1f} us per client-step", flush=True)
    c.close()
wl = synth.preset("C5")
sizes = synth.client_sizes(wl)
cohort = synth.cohort(wl)
_, x, y = synth.population(wl, sizes)
th = synth.init_params("lstm")
cfg = fl.Config(model="lstm", batch_size=4, local_epochs=1, lr=wl.lr, shuffle=wl.shuffle, seed=wl.seed)
c = fl.fl_round_init(cfg, sizes, torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), th)
st = c.fl_round(cohort, round_index=0)
st = c.fl_round(cohort, round_index=1)
print(f"C5 round: {st['round_ms']:.1f} ms, waves {st['waves']}, client-steps {st['steps_local']}, "
      f"max client steps {int(np.ceil(sizes[cohort].max() / 4))}", flush=True)
