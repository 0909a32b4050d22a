"""Pins for the oracle's local SGD ("trained ... using SGD",
P:362-363 epochs of m batches; readings A4, A5, A8-A13).

Independent witnesses:
* torch CPU fp64 autograd (nn.functional conv2d / max_pool2d / linear /
  lstm, cross_entropy) driven through the same batch schedule;
* central finite differences of the loss on random coordinates;
* closed forms: lr = 0 leaves θ unchanged; B ≥ n gives full-batch GD.
"""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle
import synth



def split(model, theta):
    out, o = {}, 0
    for name, shape in synth.param_shapes(model):
        n = int(np.prod(shape))
        out[name] = torch.tensor(theta[o:o + n].reshape(shape), dtype=torch.float64, requires_grad=True)
        o += n
    return out


def flat(model, params):
    return np.concatenate([params[n].detach().numpy().ravel() for n, _ in synth.param_shapes(model)])


def torch_loss(model, p, x, y):
    """Mean CE over the batch — torch's own modules, canonical layouts."""
    y = torch.as_tensor(np.asarray(y), dtype=torch.long)
    if model == "logreg":
        z = F.linear(torch.as_tensor(x, dtype=torch.float64), p["fc.w"], p["fc.b"])
    elif model in ("cnn", "speech"):
        shape = (-1, 3, 32, 32) if model == "cnn" else (-1, 1, 40, 98)
        h = torch.as_tensor(x, dtype=torch.float64).reshape(shape)
        h = F.max_pool2d(F.relu(F.conv2d(h, p["conv1.w"], p["conv1.b"], padding=2)), 2)
        h = F.max_pool2d(F.relu(F.conv2d(h, p["conv2.w"], p["conv2.b"], padding=2)), 2)
        h = F.relu(F.linear(h.flatten(1), p["fc1.w"], p["fc1.b"]))
        z = F.linear(h, p["fc2.w"], p["fc2.b"])
    else:
        e = F.embedding(torch.as_tensor(x, dtype=torch.long), p["emb"])
        # torch's fused LSTM op on our parameter tensors (gate order i,f,g,o)
        out = torch._VF.lstm(e, (torch.zeros(2, e.shape[0], 256, dtype=torch.float64), torch.zeros(2, e.shape[0], 256, dtype=torch.float64)),
                             [p["w_ih_l0"], p["w_hh_l0"], p["b_ih_l0"], p["b_hh_l0"],
                              p["w_ih_l1"], p["w_hh_l1"], p["b_ih_l1"], p["b_hh_l1"]],
                             True, 2, 0.0, False, False, True)[0]
        z = F.linear(out[:, -1], p["fc.w"], p["fc.b"])
    return F.cross_entropy(z, y)


def torch_local_sgd(model, theta, x, y, B, E, lr, perms=None):
    p = split(model, theta)
    n = len(y)
    for e in range(E):
        pi = np.arange(n) if perms is None else perms[e]
        for j in range(-(-n // B)):
            b = pi[j * B:min((j + 1) * B, n)]
            loss = torch_loss(model, p, x[b], y[b])
            grads = torch.autograd.grad(loss, list(p.values()))
            with torch.no_grad():
                for t, g in zip(p.values(), grads):
                    t -= lr * g
    return flat(model, p)


def data(model, n, seed=0):
    wl = synth.preset({"logreg": "C1", "cnn": "C2", "speech": "C4", "lstm": "C5"}[model])
    x, y = synth.client_data(wl, seed, n)
    return x, y


def test_param_counts_match_paper_appendix():
    """McMahan CNN 'same' padding on CIFAR = 2,156,490 (reading A10)."""
    assert oracle.n_params("cnn") == 2_156_490 == synth.n_params("cnn")
    assert oracle.n_params("speech") == 3_993_507 == synth.n_params("speech")
    assert oracle.n_params("lstm") == 819_920 == synth.n_params("lstm")
    assert oracle.n_params("logreg") == 7_850 == synth.n_params("logreg")


@pytest.mark.parametrize("model,n,B,E,lr", [("logreg", 13, 5, 2, 0.1), ("cnn", 5, 2, 2, 0.05),
                                            ("speech", 3, 2, 1, 0.05), ("lstm", 3, 2, 1, 0.5)])
def test_local_sgd_matches_torch_autograd(model, n, B, E, lr):
    theta = synth.init_params(model).astype(np.float64)
    x, y = data(model, n)
    ours = oracle.local_sgd(model, theta, x, y, B, E, lr)
    ref = torch_local_sgd(model, theta, x, y, B, E, lr)
    assert np.max(np.abs(ours - ref)) < 1e-10
    assert np.max(np.abs(ours - theta)) > 1e-4  # something actually moved


def test_shuffled_schedule_matches_torch():
    model, n, B, E, lr = "cnn", 6, 4, 2, 0.05
    theta = synth.init_params(model).astype(np.float64)
    x, y = data(model, n, seed=3)
    perms = [oracle.perm(42, 1, 3, e, n) for e in range(E)]
    ours = oracle.local_sgd(model, theta, x, y, B, E, lr, shuffle=1, seed=42, rnd=1, cid=3)
    ref = torch_local_sgd(model, theta, x, y, B, E, lr, perms=perms)
    assert np.max(np.abs(ours - ref)) < 1e-10


@pytest.mark.parametrize("model", ["logreg", "cnn", "speech", "lstm"])
def test_gradient_finite_differences(model):
    rng = np.random.default_rng(1)
    theta = synth.init_params(model).astype(np.float64)
    x, y = data(model, 1, seed=2)
    _, g = oracle.sample_grad(model, theta, x[0], int(y[0]))
    P = theta.size
    idx = rng.choice(P, size=6, replace=False)
    idx = np.concatenate([idx, np.argsort(-np.abs(g))[:4]])  # include the largest entries
    h = 1e-6
    for i in idx:
        tp, tm = theta.copy(), theta.copy()
        tp[i] += h
        tm[i] -= h
        fd = (oracle.sample_grad(model, tp, x[0], int(y[0]))[0] - oracle.sample_grad(model, tm, x[0], int(y[0]))[0]) / (2 * h)
        assert abs(fd - g[i]) <= 1e-6 + 1e-5 * abs(g[i]), (model, i, fd, g[i])


@pytest.mark.parametrize("model", ["logreg", "cnn"])
def test_lr_zero_leaves_model_unchanged(model):
    theta = synth.init_params(model).astype(np.float64)
    x, y = data(model, 7)
    out = oracle.local_sgd(model, theta, x, y, 3, 2, 0.0)
    assert np.array_equal(out, theta)


def test_full_batch_is_gradient_descent():
    """B ≥ n: each epoch is one full-batch GD step on the mean loss."""
    model = "logreg"
    theta = synth.init_params(model).astype(np.float64)
    x, y = data(model, 9)
    out = oracle.local_sgd(model, theta, x, y, 100, 3, 0.1)
    ref = torch_local_sgd(model, theta, x, y, 9, 3, 0.1)
    assert np.max(np.abs(out - ref)) < 1e-12


def test_logreg_hand_case():
    """n=1, 2 nonzero features, zero init: z = b = 0 ⇒ p = 1/10, so
    ∇W[q] = (0.1 − [q=y]) x and ∇b[q] = 0.1 − [q=y] (textbook softmax-CE)."""
    theta = np.zeros(7850)
    x = np.zeros((1, 784), dtype=np.float32)
    x[0, 0], x[0, 1] = 2.0, -1.0
    loss, g = oracle.sample_grad("logreg", theta, x[0], 3)
    assert loss == pytest.approx(np.log(10.0), rel=1e-15)
    W = g[:7840].reshape(10, 784)
    for q in range(10):
        t = 0.1 - (1.0 if q == 3 else 0.0)
        assert W[q, 0] == pytest.approx(2 * t, abs=1e-15)
        assert W[q, 1] == pytest.approx(-t, abs=1e-15)
        assert g[7840 + q] == pytest.approx(t, abs=1e-15)
    assert np.all(W[:, 2:] == 0)


def test_round_identical_clients_equal_single_client():
    """North star: identical clients ⇒ FedAvg = a single client's update."""
    wl = synth.preset("C1", n_pop=4, n_cohort=4)
    x1, y1 = synth.client_data(wl, 0, 10)
    x = np.concatenate([x1] * 4)
    y = np.concatenate([y1] * 4)
    sizes = np.array([10] * 4)
    theta = synth.init_params("logreg")
    out, N, tk = oracle.fedavg_round("logreg", theta, x, y, sizes, np.arange(4), 5, 1, 0.1)
    single = oracle.local_sgd("logreg", theta, x1, y1, 5, 1, 0.1)
    assert N == 40
    assert np.allclose(out, single, rtol=0, atol=1e-15)


def test_c3_drift_envelope_golden_matches_workload():
    """tests/golden/c3_drift_envelope.json (written by scripts/drift_envelope.py from oracle/
    only) must describe the 4 largest clients of the C3 cohort the GPU test checks, and its
    envelopes must be ordered as the precisions are (one fp32 roundoff < one TF32 rounding)."""
    import json
    import os

    import synth

    env = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "c3_drift_envelope.json")))
    wl = synth.preset("C3")
    sizes = synth.client_sizes(wl)[np.sort(synth.cohort(wl))]
    big = np.argsort(-sizes, kind="stable")[:4]
    assert env["clients"] == [int(c) for c in big] and env["sizes"] == [int(sizes[c]) for c in big]
    assert 0 < max(env["drift_fp32"]) < max(env["drift_tf32"]) < max(env["update_maxabs"])
