"""Layer-level checks of the tensor-core (tcgen05, TF32) kernels.

After one SGD wave of a client from θ_g, each tensor-core layer's output is compared
with a plain torch CPU fp64 reference of the same op applied to THAT kernel's own
inputs (read back with fl_debug_read), so upstream differences cannot mask or fake
an error.  TF32 operands keep 10 mantissa bits: outputs match to ~1e-3 relative in
norm; pooling argmax may flip only where two window values are that close.
"""
import os

import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.nn.functional as F  # noqa: E402

import paper_2306_17453_b200 as fl  # noqa: E402

B = 32
TOL = 4e-3  # relative Frobenius error allowed for TF32 tensor-core outputs


def params(theta):
    out, o = {}, 0
    for n, s in synth.param_shapes("cnn"):
        k = int(np.prod(s))
        out[n] = torch.tensor(theta[o:o + k].reshape(s), dtype=torch.float64)
        o += k
    return out


def one_wave(sizes, math=0):
    wl = synth.preset("C2", n_pop=len(sizes), n_cohort=len(sizes))
    _, x, y = synth.population(wl, sizes)
    theta = synth.init_params("cnn")
    cfg = fl.Config(model="cnn", batch_size=B, lr=wl.lr, math=math)
    # one client group, no solo streams: client a's wave-0 activations sit at slots [a·B, a·B + B)
    # of the debug buffers (the scheduler otherwise spreads clients over per-group buffers)
    saved = {k: os.environ.get(k) for k in ("FL_GROUPS", "FL_SOLO")}
    os.environ.update(FL_GROUPS="1", FL_SOLO="0")
    try:
        ctx = fl.fl_round_init(cfg, sizes, torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda(), theta)
    finally:
        for k, v in saved.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    ctx.fl_place(np.arange(len(sizes)))
    ctx.fl_train_clients(0)  # single-step clients: the buffers hold wave 0
    return ctx, theta


def nchw(a):  # [S][H][W][C] -> torch [S][C][H][W] fp64
    return torch.from_numpy(np.ascontiguousarray(a)).double().permute(0, 3, 1, 2)


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-30))


SIZES = [np.array([32]), np.array([32, 5, 17])]
# conv1's kernels split a wave's half-sample tiles evenly over the CTAs, so with more tiles than
# SMs one CTA's range crosses client boundaries (rebuilding the shifted taps in TMEM, closing a dW
# segment mid-range): 40 clients, ragged ones in between
SIZES_MANY = [np.array([32] * 12 + [7] + [32] * 12 + [19, 3] + [32] * 12 + [30])]


@pytest.mark.parametrize("sizes", SIZES)
def test_conv2_forward_pool_tc(sizes):
    ctx, theta = one_wave(sizes)
    S = len(sizes) * B
    p1 = ctx.fl_debug_read("p1", (S, 16, 16, 32))
    p2 = ctx.fl_debug_read("p2", (S, 8, 8, 64))
    am2 = ctx.fl_debug_read("am2", (S, 8, 8, 64), np.uint8)
    P = params(theta)
    valid = np.concatenate([np.arange(a * B, a * B + int(n)) for a, n in enumerate(sizes)])
    a2 = F.conv2d(nchw(p1[valid]), P["conv2.w"], P["conv2.b"], padding=2)
    ref, idx = F.max_pool2d(F.relu(a2), 2, return_indices=True)
    ref = ref.permute(0, 2, 3, 1).numpy()
    assert rel(p2[valid], ref) < TOL
    # argmax: torch's flat index over the 16x16 plane -> window position (di*2 + dj)
    idx = idx.permute(0, 2, 3, 1).numpy()
    di, dj = (idx // 16) % 2, (idx % 16) % 2
    pos = di * 2 + dj
    positive = ref > 1e-3 * np.abs(ref).max()  # windows with a ReLU-active maximum
    assert np.mean(am2[valid][positive] == pos[positive]) > 0.995


def unpool_ref(dp, p, am):
    """pool backward (reading A13): route dp to the argmax of each 2x2 window if p > 0."""
    g = np.where(p > 0, dp, 0.0)
    out = np.zeros((len(dp), 2 * dp.shape[1], 2 * dp.shape[2], dp.shape[3]))
    for t in range(4):
        di, dj = divmod(t, 2)
        out[:, di::2, dj::2, :] = np.where(am == t, g, 0.0)
    return out


@pytest.mark.parametrize("sizes", SIZES)
def test_conv2_dx_pool1_relu_tc(sizes):
    ctx, theta = one_wave(sizes)
    S = len(sizes) * B
    dY2 = ctx.fl_debug_read("dY2", (S, 16, 16, 64))
    p1 = ctx.fl_debug_read("p1", (S, 16, 16, 32))
    dp1m = ctx.fl_debug_read("dp1", (S, 16, 16, 32))  # conv2 dX with pool1's ReLU' (routing is in conv1 dW)
    P = params(theta)
    valid = np.concatenate([np.arange(a * B, a * B + int(n)) for a, n in enumerate(sizes)])
    dp1 = F.conv_transpose2d(nchw(dY2[valid]), P["conv2.w"], padding=2).permute(0, 2, 3, 1).numpy()
    assert rel(dp1m[valid], np.where(p1[valid] > 0, dp1, 0.0)) < TOL


def _grad_from_update(ctx, theta, client, lr):
    """(θ_g − θ_k)/η for a single-step client = its mean gradient (canonical layout)."""
    return params((theta.astype(np.float64) - ctx.fl_get_client_params(client).astype(np.float64)) / lr)


@pytest.mark.parametrize("sizes", SIZES)
def test_conv2_dw_tc(sizes):
    ctx, theta = one_wave(sizes)
    S = len(sizes) * B
    p1 = ctx.fl_debug_read("p1", (S, 16, 16, 32))
    dY2 = ctx.fl_debug_read("dY2", (S, 16, 16, 64))
    lr = synth.preset("C2").lr
    for a, n in enumerate(sizes):
        rows = slice(a * B, a * B + int(n))
        g = _grad_from_update(ctx, theta, a, lr)
        dy = nchw(dY2[rows])
        ref_w = torch.nn.grad.conv2d_weight(nchw(p1[rows]), (64, 32, 5, 5), dy, padding=2).numpy()
        ref_b = dy.sum((0, 2, 3)).numpy()
        assert rel(g["conv2.w"].numpy(), ref_w) < TOL, a
        assert rel(g["conv2.b"].numpy(), ref_b) < TOL, a


def client_x(sizes):
    wl = synth.preset("C2", n_pop=len(sizes), n_cohort=len(sizes))
    _, x, _ = synth.population(wl, sizes)
    off = np.concatenate([[0], np.cumsum(sizes)])
    return [torch.from_numpy(x[off[a]:off[a + 1]]).double().reshape(-1, 3, 32, 32) for a in range(len(sizes))]


@pytest.mark.parametrize("sizes", SIZES + SIZES_MANY)
def test_conv1_forward_tc(sizes):
    ctx, theta = one_wave(sizes)
    S = len(sizes) * B
    p1 = ctx.fl_debug_read("p1", (S, 16, 16, 32))
    am1 = ctx.fl_debug_read("am1", (S, 16, 16, 32), np.uint8)
    P = params(theta)
    for a, xa in enumerate(client_x(sizes)):
        pre = F.conv2d(xa, P["conv1.w"], P["conv1.b"], padding=2)  # [n][32][32][32] fp64
        ref = F.max_pool2d(F.relu(pre), 2)
        assert rel(p1[a * B:a * B + len(xa)], ref.permute(0, 2, 3, 1).numpy()) < TOL, a
        # pool1's argmax (row-major window index) must select a maximum of its window, up to
        # TF32 rounding of near-ties
        win = pre.numpy().reshape(len(xa), 32, 16, 2, 16, 2).transpose(0, 2, 4, 1, 3, 5).reshape(len(xa), 16, 16, 32, 4)
        am = am1[a * B:a * B + len(xa)].astype(np.int64)
        assert am.max() <= 3
        picked = np.take_along_axis(win, am[..., None], axis=-1)[..., 0]
        gap = win.max(-1) - picked
        assert gap.max() <= 1e-3 * np.abs(win).max(), (a, float(gap.max()))


@pytest.mark.parametrize("sizes", SIZES + SIZES_MANY)
def test_conv1_dw_tc(sizes):
    ctx, theta = one_wave(sizes)
    S = len(sizes) * B
    # dY1 never reaches HBM: the kernel expands it from dp1m and pool1's argmax on chip, so the
    # reference expands the same inputs with the plain pool-backward definition
    p1 = ctx.fl_debug_read("p1", (S, 16, 16, 32))
    am1 = ctx.fl_debug_read("am1", (S, 16, 16, 32), np.uint8)
    dp1m = ctx.fl_debug_read("dp1", (S, 16, 16, 32))
    dY1 = unpool_ref(dp1m, p1, am1)
    lr = synth.preset("C2").lr
    for a, xa in enumerate(client_x(sizes)):
        g = _grad_from_update(ctx, theta, a, lr)
        dy = nchw(dY1[a * B:a * B + len(xa)])
        ref_w = torch.nn.grad.conv2d_weight(xa, (32, 3, 5, 5), dy, padding=2).numpy()
        assert rel(g["conv1.w"].numpy(), ref_w) < TOL, a
        assert rel(g["conv1.b"].numpy(), dy.sum((0, 2, 3)).numpy()) < TOL, a


def p2_canonical(p2):  # [S][8][8][64] (h, w, c) -> [S][4096] in torch's (c, h, w) flatten order
    return torch.from_numpy(np.ascontiguousarray(p2)).double().permute(0, 3, 1, 2).reshape(len(p2), -1)


@pytest.mark.parametrize("sizes", SIZES)
def test_fc1_forward_tc(sizes):
    ctx, theta = one_wave(sizes)
    S = len(sizes) * B
    p2 = ctx.fl_debug_read("p2", (S, 8, 8, 64))
    h = ctx.fl_debug_read("h", (S, 512))
    P = params(theta)
    for a, n in enumerate(sizes):
        rows = slice(a * B, a * B + int(n))
        ref = F.relu(F.linear(p2_canonical(p2[rows]), P["fc1.w"], P["fc1.b"])).numpy()
        assert rel(h[rows], ref) < TOL, a


@pytest.mark.parametrize("sizes", SIZES)
def test_fc1_dx_pool_backward_tc(sizes):
    ctx, theta = one_wave(sizes)
    S = len(sizes) * B
    p2 = ctx.fl_debug_read("p2", (S, 8, 8, 64))
    am2 = ctx.fl_debug_read("am2", (S, 8, 8, 64), np.uint8)
    dh = ctx.fl_debug_read("dh", (S, 512))
    dY2 = ctx.fl_debug_read("dY2", (S, 16, 16, 64))
    P = params(theta)
    for a, n in enumerate(sizes):
        rows = slice(a * B, a * B + int(n))
        dp2 = (torch.from_numpy(dh[rows]).double() @ P["fc1.w"]).reshape(-1, 64, 8, 8).permute(0, 2, 3, 1).numpy()
        dp2 = np.where(p2[rows] > 0, dp2, 0.0)  # ReLU' of the pooled maximum
        ref = np.zeros((int(n), 16, 16, 64))
        for t in range(4):  # window position (di, dj) = divmod(t, 2), reading A13 order
            di, dj = divmod(t, 2)
            ref[:, di::2, dj::2, :] = np.where(am2[rows] == t, dp2, 0.0)
        assert rel(dY2[rows], ref) < TOL, a


@pytest.mark.parametrize("sizes", SIZES)
def test_fc1_dw_sgd_tc(sizes):
    ctx, theta = one_wave(sizes)
    S = len(sizes) * B
    p2 = ctx.fl_debug_read("p2", (S, 8, 8, 64))
    dh = ctx.fl_debug_read("dh", (S, 512))
    lr = synth.preset("C2").lr
    for a, n in enumerate(sizes):
        rows = slice(a * B, a * B + int(n))
        g = _grad_from_update(ctx, theta, a, lr)
        dhr = torch.from_numpy(dh[rows]).double()
        assert rel(g["fc1.w"].numpy(), (dhr.T @ p2_canonical(p2[rows])).numpy()) < TOL, a
        assert rel(g["fc1.b"].numpy(), dhr.sum(0).numpy()) < TOL, a


def test_tc_path_close_to_fp32_path():
    """Whole wave: tensor-core path vs FP32 SIMT path on the same client (drift only)."""
    ctx0, _ = one_wave(np.array([32]), 0)
    ctx1, _ = one_wave(np.array([32]), 1)
    for k, shp in [("p2", (32, 8, 8, 64)), ("h", (32, 512))]:
        assert rel(ctx0.fl_debug_read(k, shp), ctx1.fl_debug_read(k, shp)) < TOL
