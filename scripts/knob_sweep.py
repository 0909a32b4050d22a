"""Median device round time of C2 (and a 400-client C3-law cohort, E=1) under env knob settings.
usage: knob_sweep.py "FL_DW2_MINS=2 FL_DW1_MINR=32" "..."   (each arg = one setting, run in a subprocess)"""
import json, os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if os.environ.get("_KNOB_CHILD"):
    import numpy as np, torch, statistics
    import synth, paper_2306_17453_b200 as fl
    out = {}
    sets = os.environ.get("KNOB_SETS", "C2,C3x400").split(",")
    cfgs = {"C2": synth.preset("C2"), "C3x400": synth.preset("C3", n_pop=400, n_cohort=400, E=1), "C3": synth.preset("C3")}
    for name in sets:
        wl = cfgs[name]
        if name == "C3":  # the bench workload: the cohort's 1,000 clients of the 10,000 population
            sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
            from bench import pop_for
            sizes, x, y, _ = pop_for(wl)
        else:
            sizes = synth.client_sizes(wl)
            _, x, y = synth.population(wl, sizes)
        ctx = fl.fl_round_init(fl.Config(model="cnn", batch_size=32, local_epochs=wl.E, lr=wl.lr), sizes, torch.from_numpy(x).cuda(),
                               torch.from_numpy(y).cuda(), synth.init_params("cnn"))
        ids = np.arange(len(sizes))
        for i in range(3):
            ctx.fl_round(ids, round_index=i, stats=False)
        out[name] = statistics.median(ctx.fl_round(ids, round_index=3 + i)["round_ms"] for i in range(8))
        ctx.close()
        del x, y
    print(json.dumps(out))
    sys.exit(0)
for setting in sys.argv[1:] or [""]:
    env = dict(os.environ, _KNOB_CHILD="1")
    for kv in setting.split():
        k, v = kv.split("=")
        env[k] = v
    r = subprocess.run([sys.executable, __file__], env=env, capture_output=True, text=True)
    print(f"{setting or 'default':50s} {r.stdout.strip() or r.stderr[-300:]}", flush=True)
