"""Drift envelope of the C3 long-trajectory parity check (reading R14), from the
fp64 oracle alone: how far two EXACT (fp64) local-SGD trajectories of the 4 largest C3 clients
(126 steps each, E = 2) end up apart when θ_g is perturbed ONCE before training: rounded to
TF32 (10-bit mantissa), or moved by one fp32 unit roundoff (each element times 1 ± 2^-24,
seeded signs).  A GPU path that rounds at every operation cannot be expected closer to the
fp64 trajectory than the problem's own sensitivity to one such rounding; the test bounds
each path's drift by twice the envelope of its precision.

Calls only oracle/ and synth/ (test infrastructure); writes tests/golden/c3_drift_envelope.json.
usage: python scripts/drift_envelope.py  (~15 min on 8 host cores)"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import synth  # noqa: E402


def round_tf32(a):
    """Round-to-nearest to 10 explicit mantissa bits (the TF32 operand precision)."""
    b = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)
    b = ((b + np.uint32(0x1000)) & np.uint32(0xFFFFE000)).astype(np.uint32)
    return b.view(np.float32).astype(np.float64)


def main():
    wl = synth.preset("C3")
    sizes_all = synth.client_sizes(wl)
    ids = np.sort(synth.cohort(wl))
    _, x, y = synth.population(wl, sizes_all, clients=ids)
    sizes = sizes_all[ids]
    theta = synth.init_params("cnn")
    big = np.argsort(-sizes, kind="stable")[:4]
    off = np.concatenate([[0], np.cumsum(sizes)])
    t0 = time.time()
    ref, _ = oracle.train_clients("cnn", theta, x, y, off, big, wl.B, wl.E, wl.lr)
    out = {"clients": [int(c) for c in big], "sizes": [int(sizes[c]) for c in big],
           "update_maxabs": [float(np.max(np.abs(ref[i] - theta))) for i in range(4)]}
    sign = np.random.default_rng(7).choice([-1.0, 1.0], size=theta.shape)
    for name, th in (("tf32", round_tf32(theta)), ("fp32", theta * (1.0 + sign * 2.0 ** -24))):
        alt, _ = oracle.train_clients("cnn", th, x, y, off, big, wl.B, wl.E, wl.lr)
        out["drift_" + name] = [float(np.max(np.abs(alt[i] - ref[i]))) for i in range(4)]
        print(name, out["drift_" + name], flush=True)
    out["seconds"] = round(time.time() - t0, 1)
    out["how"] = ("scripts/drift_envelope.py: max-abs distance after E = 2 epochs between fp64 oracle "
                  "trajectories from theta_g and from theta_g rounded once to tf32 / perturbed by one fp32 roundoff")
    path = os.path.join(ROOT, "tests", "golden", "c3_drift_envelope.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
