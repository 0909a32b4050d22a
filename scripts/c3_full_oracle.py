"""North-star parity at full size: one C3 round (1,000 of 10,000 CIFAR-shaped clients, E = 2,
B = 32) on the GPU (TF32 tensor-core path) against the fp64 oracle run over EVERY client on the
host cores (minutes).  Reports max-abs |θ_new,GPU − θ_new,oracle| (the north-star 1e-3 bar),
the per-client θ_k errors, and, for the 4 largest clients, the FP32 SIMT path (math = 1) against
the oracle (separates TF32 drift from kernel logic).  Output: gpurun_out/c3_parity.json."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, synth, paper_2306_17453_b200 as fl

wl = synth.preset("C3")
sizes_all = synth.client_sizes(wl)
ids = np.sort(synth.cohort(wl))
_, x, y = synth.population(wl, sizes_all, clients=ids)
sizes = sizes_all[ids]
theta = synth.init_params("cnn")
xd, yd = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
res = {"workload": "C3: 1,000 of 10,000 CIFAR-shaped clients, E=2, B=32, lr=%g" % wl.lr}
cohort = np.arange(len(ids))
order = np.argsort(-sizes, kind="stable")
big = order[:4]
# FP32 SIMT path (math = 1) for the 4 largest clients
ctx = fl.fl_round_init(fl.Config(model="cnn", batch_size=wl.B, local_epochs=wl.E, lr=wl.lr, math=1), sizes, xd, yd,
                       theta)
ctx.fl_place(big)
ctx.fl_train_clients(0)
tk_simt = np.stack([ctx.fl_get_client_params(c) for c in big])
ctx.close()
# the TF32 round (the product path), kept alive so each θ_k can be fetched after aggregation
ctx = fl.fl_round_init(fl.Config(model="cnn", batch_size=wl.B, local_epochs=wl.E, lr=wl.lr), sizes, xd, yd, theta)
ctx.fl_place(cohort)
ctx.fl_train_clients(0)
out, N = ctx.fl_aggregate()
# oracle over every client, in chunks of similar sizes (largest first); Σ n_k θ_k in fp64
pop_off = np.concatenate([[0], np.cumsum(sizes)])
S = np.zeros(len(theta))
e_k = np.zeros(len(cohort))
t0 = time.time()
CH = 32
simt_err = []
for s0 in range(0, len(order), CH):
    chunk = order[s0:s0 + CH]
    tk_ref, used = oracle.train_clients("cnn", theta, x, y, pop_off, chunk, wl.B, wl.E, wl.lr)
    for j, c in enumerate(chunk):
        S += float(sizes[c]) * tk_ref[j]
        e_k[c] = np.max(np.abs(ctx.fl_get_client_params(c) - tk_ref[j]))
        if s0 == 0 and j < 4:
            simt_err.append(float(np.max(np.abs(tk_simt[j] - tk_ref[j]))))
    print("oracle chunk", s0, "%.0f s" % (time.time() - t0), flush=True)
res["oracle_seconds"], res["oracle_threads"] = time.time() - t0, used
ref_new = S / float(sizes.sum())
assert int(sizes.sum()) == N
e_new = np.abs(out.astype(np.float64) - ref_new)
res.update({
    "theta_new_maxabs_err": float(e_new.max()), "theta_new_mean_abs_err": float(e_new.mean()),
    "theta_new_tolerance": 1e-3,
    "theta_k_err_quantiles_p50_p90_p99_max": [float(np.percentile(e_k, q)) for q in (50, 90, 99, 100)],
    "theta_k_err_largest4": [float(e_k[i]) for i in big], "sizes_largest4": sizes[big].tolist(),
    "simt_fp32_err_largest4": simt_err,
    "clients_over_1e-3": int((e_k > 1e-3).sum()),
})
os.makedirs("gpurun_out", exist_ok=True)
json.dump(res, open("gpurun_out/c3_parity.json", "w"), indent=1)
print(json.dumps(res, indent=1))
