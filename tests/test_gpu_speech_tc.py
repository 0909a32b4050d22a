"""Layer-level checks of the speech CNN (C4 shapes: 1x40x98 input, conv2 on a 20x49 plane,
fc1 15,360 -> 256, batch 20 in 32-row slots) on the tensor-core path (math = 0).

conv2 (forward + pool, dX, dW) runs the patched tcgen05 kernels (8x16 patches, TMA zero fill
past the image) and fc1 the tcgen05 forward / fused backward with the odd 49th column of the
conv2 plane receiving no gradient (floor pooling).  Each layer's output after one SGD wave is
compared with a torch CPU fp64 reference of the same op on that kernel's own inputs (read
back with fl_debug_read), as in test_gpu_kernels.py; TF32 operands -> ~1e-3 relative.
"""
import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.nn.functional as F  # noqa: E402

import paper_2306_17453_b200 as fl  # noqa: E402

BP = 32          # slot pitch of the tensor-core path
TOL = 4e-3       # relative Frobenius error of TF32 outputs
SIZES = np.array([20, 7, 13], dtype=np.int64)  # one SGD step each (B = 20)


def params(theta):
    out, o = {}, 0
    for n, s in synth.param_shapes("speech"):
        k = int(np.prod(s))
        out[n] = torch.tensor(theta[o:o + k].reshape(s), dtype=torch.float64)
        o += k
    return out


def nchw(a):
    return torch.from_numpy(np.ascontiguousarray(a)).double().permute(0, 3, 1, 2)


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-30))


@pytest.fixture(scope="module")
def wave():
    wl = synth.preset("C4", n_pop=len(SIZES), n_cohort=len(SIZES))
    _, x, y = synth.population(wl, SIZES)
    theta = synth.init_params("speech")
    cfg = fl.Config(model="speech", batch_size=wl.B, lr=wl.lr)
    ctx = fl.fl_round_init(cfg, SIZES, torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), theta)
    ctx.fl_place(np.arange(len(SIZES)))
    ctx.fl_train_clients(0)
    S = len(SIZES) * BP
    valid = np.concatenate([np.arange(a * BP, a * BP + int(n)) for a, n in enumerate(SIZES)])
    yield ctx, theta, S, valid, wl.lr
    ctx.close()


def test_speech_conv2_forward_pool_tc(wave):
    ctx, theta, S, valid, _ = wave
    p1 = ctx.fl_debug_read("p1", (S, 20, 49, 32))
    p2 = ctx.fl_debug_read("p2", (S, 10, 24, 64))
    am2 = ctx.fl_debug_read("am2", (S, 10, 24, 64), np.uint8)
    P = params(theta)
    a2 = F.conv2d(nchw(p1[valid]), P["conv2.w"], P["conv2.b"], padding=2)
    ref, idx = F.max_pool2d(F.relu(a2), 2, return_indices=True)  # floor: the 49th column is dropped
    ref = ref.permute(0, 2, 3, 1).numpy()
    assert rel(p2[valid], ref) < TOL
    idx = idx.permute(0, 2, 3, 1).numpy()
    pos = ((idx // 49) % 2) * 2 + (idx % 49) % 2
    positive = ref > 1e-3 * np.abs(ref).max()
    assert np.mean(am2[valid][positive] == pos[positive]) > 0.995


def test_speech_fc1_backward_dY2_tc(wave):
    """fused fc1 dX -> pool2 / ReLU backward -> dY2 on the 20 x 49 plane (column 48 gets none)."""
    ctx, theta, S, valid, _ = wave
    dh = ctx.fl_debug_read("dh", (S, 256))
    p2 = ctx.fl_debug_read("p2", (S, 10, 24, 64))
    am2 = ctx.fl_debug_read("am2", (S, 10, 24, 64), np.uint8)
    dY2 = ctx.fl_debug_read("dY2", (S, 20, 49, 64))
    P = params(theta)
    dp2 = (torch.from_numpy(dh[valid]).double() @ P["fc1.w"]).reshape(-1, 64, 10, 24).permute(0, 2, 3, 1).numpy()
    g = np.where(p2[valid] > 0, dp2, 0.0)
    ref = np.zeros((len(valid), 20, 49, 64))
    for t in range(4):
        di, dj = divmod(t, 2)
        ref[:, di:20:2, dj:48:2, :] = np.where(am2[valid] == t, g, 0.0)
    assert rel(dY2[valid], ref) < TOL
    assert np.all(dY2[valid][:, :, 48, :] == 0.0)


def test_speech_conv2_dx_tc(wave):
    ctx, theta, S, valid, _ = wave
    dY2 = ctx.fl_debug_read("dY2", (S, 20, 49, 64))
    p1 = ctx.fl_debug_read("p1", (S, 20, 49, 32))
    dp1m = ctx.fl_debug_read("dp1", (S, 20, 49, 32))
    P = params(theta)
    dp1 = F.conv_transpose2d(nchw(dY2[valid]), P["conv2.w"], padding=2).permute(0, 2, 3, 1).numpy()
    assert rel(dp1m[valid], np.where(p1[valid] > 0, dp1, 0.0)) < TOL


def test_speech_conv2_dw_and_fc1_dw_tc(wave):
    """single-step clients: (θ_g − θ_k)/η is the client's gradient; conv2 dW from the
    tensor-core dW + split-K reduction, fc1 dW from the fused backward's epilogue."""
    ctx, theta, S, valid, lr = wave
    p1 = ctx.fl_debug_read("p1", (S, 20, 49, 32))
    dY2 = ctx.fl_debug_read("dY2", (S, 20, 49, 64))
    dh = ctx.fl_debug_read("dh", (S, 256))
    p2 = ctx.fl_debug_read("p2", (S, 10, 24, 64))
    for a, n in enumerate(SIZES):
        rows = slice(a * BP, a * BP + int(n))
        g = params((theta.astype(np.float64) - ctx.fl_get_client_params(a).astype(np.float64)) / lr)
        dy = nchw(dY2[rows])
        ref_w = torch.nn.grad.conv2d_weight(nchw(p1[rows]), (64, 32, 5, 5), dy, padding=2).numpy()
        assert rel(g["conv2.w"].numpy(), ref_w) < TOL, a
        assert rel(g["conv2.b"].numpy(), dy.sum((0, 2, 3)).numpy()) < TOL, a
        p2c = torch.from_numpy(p2[rows]).double().permute(0, 3, 1, 2).reshape(int(n), -1)  # canonical (c,h,w)
        ref_f = (torch.from_numpy(dh[rows]).double().T @ p2c).numpy()
        assert rel(g["fc1.w"].numpy(), ref_f) < TOL, a
        assert rel(g["fc1.b"].numpy(), dh[rows].sum(0)) < TOL, a
