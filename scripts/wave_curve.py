"""T(A): device time of one wave of A equal clients (|b| = 32), single stream. Run with
FL_SOLO=0 FL_GROUPS=1 so all A clients share each wave. Optional arg: 'prof' for per-kernel."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, paper_2306_17453_b200 as fl

STEPS = 8
prof = len(sys.argv) > 1 and sys.argv[1] == "prof"
for A in [1, 2, 4, 8, 16, 32, 64, 100, 148]:
    sizes = np.full(A, 32 * STEPS)
    wl = synth.preset("C2", n_pop=A, n_cohort=A)
    _, x, y = synth.population(wl, sizes)
    ctx = fl.fl_round_init(fl.Config(model="cnn", batch_size=32, lr=wl.lr), sizes, torch.from_numpy(x).cuda(),
                           torch.from_numpy(y).cuda(), synth.init_params("cnn"))
    ids = np.arange(A)
    for i in range(3): ctx.fl_round(ids, round_index=i, stats=False)
    ms = np.median([ctx.fl_round(ids, round_index=3 + i)["round_ms"] for i in range(5)])
    line = f"A={A:4d} T(A)={ms / STEPS * 1e3:8.1f} us/wave  per-client {ms / STEPS * 1e3 / A:7.2f} us"
    if prof:
        ctx.fl_set_profiling(True); ctx.fl_round(ids, round_index=99)
        ks = ctx.fl_get_kernel_stats(); ctx.fl_set_profiling(False)
        line += "  | " + " ".join(f"{k[:9]}={v['ms'] / v['launches'] * 1e3:.0f}" for k, v in
                                 sorted(ks.items(), key=lambda kv: -kv[1]['ms']) if v['launches'] >= STEPS)
    print(line, flush=True)
