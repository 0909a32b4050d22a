"""Debug: TC vs SIMT path p1 against a torch reference (args: order of math modes)."""
import sys; sys.path.insert(0, "tests"); sys.path.insert(0, ".")
import numpy as np, torch, torch.nn.functional as F
from test_gpu_kernels import one_wave, rel, client_x, params
import synth
P = params(synth.init_params("cnn"))
xa = client_x(np.array([32]))[0]
ref = F.max_pool2d(F.relu(F.conv2d(xa, P["conv1.w"], P["conv1.b"], padding=2)), 2).permute(0, 2, 3, 1).numpy()
for m in [int(a) for a in sys.argv[1:]]:
    c, _ = one_wave(np.array([32]), m)
    p1 = c.fl_debug_read("p1", (32, 16, 16, 32))
    print("math", m, "vs ref", rel(p1, ref), flush=True)
