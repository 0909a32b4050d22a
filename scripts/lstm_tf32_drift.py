"""TF32 drift study for the char-LSTM's batched GEMMs (reading R15): one C5-shaped
client's local SGD (B = 4, lr = 0.5) in torch with the operands of the batched GEMMs -- layer-1
input projection, layer-1 dX, and the weight gradients of W_ih / W_hh -- rounded to TF32
(truncation, as tcgen05 kind::tf32 reads fp32 operands), everything else fp32, against fp64.
Prints max |θ − θ_fp64| after 25 / 100 / 250 / 1000 steps.  CPU only (minutes).

    python scripts/lstm_tf32_drift.py [steps]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402

torch.set_num_threads(16)
T, H, V, E = 80, 256, 80, 8


def q_rz(t):
    i = t.float().contiguous().view(torch.int32)
    return (i & ~0x1FFF).view(torch.float32).to(t.dtype)


class QMM(torch.autograd.Function):
    """y = a @ b with tf32-truncated operands in forward and in both backward GEMMs."""

    @staticmethod
    def forward(ctx, a, b, on):
        ctx.save_for_backward(a, b)
        ctx.on = on
        q = q_rz if on else (lambda t: t)
        return q(a) @ q(b)

    @staticmethod
    def backward(ctx, g):
        a, b = ctx.saved_tensors
        q = q_rz if ctx.on else (lambda t: t)
        return q(g) @ q(b).T, q(a).T @ q(g), None


def run(theta, xs, ys, dtype, tf32, steps, lr=0.5, B=4):
    p, o = {}, 0
    for n, s in synth.param_shapes("lstm"):
        k = int(np.prod(s))
        p[n] = torch.tensor(theta[o:o + k].reshape(s), dtype=dtype, requires_grad=True)
        o += k
    names = list(p)
    out = {}
    n = len(ys)
    m = -(-n // B)
    for step in range(steps):
        j = step % m
        xb = torch.tensor(xs[j * B:(j + 1) * B].astype(np.int64))
        yb = torch.tensor(ys[j * B:(j + 1) * B].astype(np.int64))
        b = len(yb)
        e = p[names[0]][xb]  # [b, T, 8]
        hs = e
        for layer in range(2):
            wih, whh, bih, bhh = (p[names[1 + 4 * layer + i]] for i in range(4))
            if layer == 1:  # batched input projection (tensor cores on the GPU path)
                xp = QMM.apply(hs.reshape(b * T, -1), wih.T, tf32).reshape(b, T, -1) + bih + bhh
            else:
                xp = hs @ wih.T + bih + bhh
            h = torch.zeros(b, H, dtype=dtype)
            c = torch.zeros(b, H, dtype=dtype)
            outs = []
            for t in range(T):
                g = xp[:, t] + h @ whh.T
                i_, f_, g_, o_ = g.chunk(4, 1)
                c = torch.sigmoid(f_) * c + torch.sigmoid(i_) * torch.tanh(g_)
                h = torch.sigmoid(o_) * torch.tanh(c)
                outs.append(h)
            hs = torch.stack(outs, 1)
        z = hs[:, -1] @ p[names[9]].T + p[names[10]]
        loss = torch.nn.functional.cross_entropy(z, yb)
        grads = torch.autograd.grad(loss, list(p.values()))
        with torch.no_grad():
            for t_, g_ in zip(p.values(), grads):
                t_ -= lr * g_
        if step + 1 in (25, 100, 250, 1000):
            out[step + 1] = np.concatenate([t_.detach().double().numpy().ravel() for t_ in p.values()])
    return out


if __name__ == "__main__":
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 250
    wl = synth.preset("C5")
    theta = synth.init_params("lstm")
    xs, ys = synth.client_data(wl, 3, 4 * 250)
    ref = run(theta, xs, ys, torch.float64, False, steps)
    f32 = run(theta, xs, ys, torch.float32, False, steps)
    t32 = run(theta, xs, ys, torch.float32, True, steps)
    for k in sorted(ref):
        print(f"steps {k:5d}: fp32 {np.max(np.abs(f32[k] - ref[k])):.2e}   tf32-GEMMs {np.max(np.abs(t32[k] - ref[k])):.2e}",
              flush=True)
