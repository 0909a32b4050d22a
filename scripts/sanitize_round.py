"""One tiny round per model through the C-ABI, for compute-sanitizer (memcheck / racecheck /
synccheck): a 4-client CIFAR CNN round (tensor-core path), a 3-client speech round, a 3-client
char-LSTM round (16-CTA cluster recurrences + tcgen05 GEMMs), a logreg round."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2306_17453_b200 as fl  # noqa: E402
import synth  # noqa: E402

which = sys.argv[1:] or ["cnn", "speech", "lstm", "logreg"]
cases = {"cnn": ("C2", [3, 33, 9, 40]), "speech": ("C4", [20, 7, 13]), "lstm": ("C5", [4, 9, 6]),
         "logreg": ("C1", [5, 12, 30])}
for name in which:
    preset, sizes = cases[name]
    sizes = np.array(sizes, dtype=np.int64)
    wl = synth.preset(preset, n_pop=len(sizes), n_cohort=len(sizes))
    _, x, y = synth.population(wl, sizes)
    cfg = fl.Config(model=wl.model, batch_size=wl.B, local_epochs=wl.E, lr=wl.lr)
    ctx = fl.fl_round_init(cfg, sizes, torch.from_numpy(x).cuda(), torch.from_numpy(y.astype(np.int32)).cuda(),
                           synth.init_params(wl.model))
    st = ctx.fl_round(np.arange(len(sizes)))
    print(name, "ok", round(st["round_ms"], 3), "ms", st["kernels"], "kernels", flush=True)
    ctx.close()
