"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds NO arithmetic of the method (no training, no averaging,
no placement).  It only draws random numbers with the shapes and
distributions of the paper's workloads (SURVEY.md §8d "Synthetic inputs"):

* client sizes: n = clamp(round(exp(mu + sigma*z)), lo, hi), z ~ N(0,1)
  (heavy-tailed, "spanning orders of magnitude", §3.1,
  Fig. 1), or Uniform{lo..hi} for config C1;
* image/speech features: class-conditional Gaussian x = mu_y + eps,
  mu_c ~ N(0, 0.25 I), eps ~ N(0, I); per-client labels
  y ~ Categorical(p_k), p_k ~ Dirichlet(0.5) (non-IID);
* Shakespeare-shaped characters: i.i.d. from a Zipf(1.1) unigram over
  80 symbols, 80 input chars + 1 target char per sample;
* initial global model theta_g: PyTorch-default U(-1/sqrt(fan_in), ..)
  per tensor, embedding N(0,1) in the canonical flat layout
  (torch state_dict order, C-contiguous).

Every draw comes from numpy PCG64 streams keyed by (master seed, stream
id, client id), so any single client's data can be regenerated alone.
Stream ids: sizes 0, cohort 1, data 2, theta_g 3, class means 4.
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace
from typing import Optional

import numpy as np

MASTER_SEED = 230617453

MODEL_IDS = {"logreg": 0, "cnn": 1, "speech": 2, "lstm": 3}


@dataclass(frozen=True)
class Workload:
    """One BASELINE.json config (or a small parity variant of one)."""
    name: str
    model: str               # logreg | cnn | speech | lstm
    n_pop: int               # population size
    n_cohort: int            # clients per round
    size_law: tuple          # ("lognormal", mu, sigma, lo, hi) | ("uniform", lo, hi)
    B: int
    E: int
    lr: float
    shuffle: int = 0
    seed: int = MASTER_SEED


# BASELINE.json configs[0..4]; unstated hyper-parameters per SURVEY §8c A7/A8.  lr of the CNN
# configs is 0.01, not A8's first guess 0.05: at 0.05 the local SGD trajectory is chaotic (an
# fp32 run departs from fp64 by 2.6e-3 after 25 steps), see DESIGN.md "Readings" R8.
PRESETS = {
    "C1": Workload("C1", "logreg", 10, 10, ("uniform", 5, 50), 5, 1, 0.1),
    "C2": Workload("C2", "cnn", 100, 100, ("lognormal", 4.952, 1.028, 10, 2000), 32, 1, 0.01),
    "C3": Workload("C3", "cnn", 10000, 1000, ("lognormal", 4.952, 1.028, 10, 2000), 32, 2, 0.01),
    "C4": Workload("C4", "speech", 2000, 2000, ("lognormal", 3.557, 1.2, 5, 5000), 20, 1, 0.01),
    "C5": Workload("C5", "lstm", 700, 700, ("lognormal", 4.840, 1.341, 4, 4000), 4, 1, 0.5),
}


def preset(name: str, **overrides) -> Workload:
    return replace(PRESETS[name], **overrides)


# ---------------------------------------------------------------- shapes
# Input-generation shape table (feature dims, classes, and parameter
# tensor shapes with their fan-in, used ONLY to draw theta_g).
FEATURES = {"logreg": 784, "cnn": 3 * 32 * 32, "speech": 1 * 40 * 98, "lstm": 80}
CLASSES = {"logreg": 10, "cnn": 10, "speech": 35, "lstm": 80}


def _param_tensors(model: str):
    """(name, shape, init) in canonical order. init = ('u', bound) | ('n',)."""
    if model == "logreg":
        return [("fc.w", (10, 784), ("u", 784 ** -0.5)), ("fc.b", (10,), ("u", 784 ** -0.5))]
    if model in ("cnn", "speech"):
        cin, hid, ncls, flat = (3, 512, 10, 64 * 8 * 8) if model == "cnn" else (1, 256, 35, 64 * 10 * 24)
        return [
            ("conv1.w", (32, cin, 5, 5), ("u", (cin * 25) ** -0.5)),
            ("conv1.b", (32,), ("u", (cin * 25) ** -0.5)),
            ("conv2.w", (64, 32, 5, 5), ("u", (32 * 25) ** -0.5)),
            ("conv2.b", (64,), ("u", (32 * 25) ** -0.5)),
            ("fc1.w", (hid, flat), ("u", flat ** -0.5)),
            ("fc1.b", (hid,), ("u", flat ** -0.5)),
            ("fc2.w", (ncls, hid), ("u", hid ** -0.5)),
            ("fc2.b", (ncls,), ("u", hid ** -0.5)),
        ]
    if model == "lstm":
        k = 256 ** -0.5
        return [
            ("emb", (80, 8), ("n",)),
            ("w_ih_l0", (1024, 8), ("u", k)), ("w_hh_l0", (1024, 256), ("u", k)),
            ("b_ih_l0", (1024,), ("u", k)), ("b_hh_l0", (1024,), ("u", k)),
            ("w_ih_l1", (1024, 256), ("u", k)), ("w_hh_l1", (1024, 256), ("u", k)),
            ("b_ih_l1", (1024,), ("u", k)), ("b_hh_l1", (1024,), ("u", k)),
            ("fc.w", (80, 256), ("u", k)), ("fc.b", (80,), ("u", k)),
        ]
    raise ValueError(model)


def param_shapes(model: str):
    return [(n, s) for n, s, _ in _param_tensors(model)]


def n_params(model: str) -> int:
    return int(sum(np.prod(s) for _, s in param_shapes(model)))


def _rng(seed: int, stream: int, key: int = 0) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64([seed & 0xFFFFFFFF, stream, key]))


# ---------------------------------------------------------------- draws
def client_sizes(wl: Workload) -> np.ndarray:
    """int64[n_pop] sample counts, client-id order."""
    rng = _rng(wl.seed, 0)
    law = wl.size_law
    if law[0] == "uniform":
        return rng.integers(law[1], law[2] + 1, size=wl.n_pop).astype(np.int64)
    _, mu, sigma, lo, hi = law
    z = rng.standard_normal(wl.n_pop)
    return np.clip(np.rint(np.exp(mu + sigma * z)), lo, hi).astype(np.int64)


def cohort(wl: Workload, round_index: int = 0) -> np.ndarray:
    """int64[n_cohort]: uniform without replacement."""
    if wl.n_cohort == wl.n_pop:
        return np.arange(wl.n_pop, dtype=np.int64)
    rng = _rng(wl.seed, 1, round_index)
    return rng.choice(wl.n_pop, size=wl.n_cohort, replace=False).astype(np.int64)


def _class_means(wl: Workload) -> np.ndarray:
    rng = _rng(wl.seed, 4)
    return (0.5 * rng.standard_normal((CLASSES[wl.model], FEATURES[wl.model]))).astype(np.float32)


_ZIPF_CACHE = {}


def _zipf_p():
    if "p" not in _ZIPF_CACHE:
        r = np.arange(1, 81, dtype=np.float64)
        p = r ** -1.1
        _ZIPF_CACHE["p"] = p / p.sum()
    return _ZIPF_CACHE["p"]


def client_data(wl: Workload, client_id: int, n: int, means: Optional[np.ndarray] = None):
    """(x, y) for one client. x: float32[n, D] (uint8[n, 80] for lstm); y: int32[n]."""
    rng = _rng(wl.seed, 2, int(client_id))
    if wl.model == "lstm":
        chars = rng.choice(80, size=(n, 81), p=_zipf_p()).astype(np.uint8)
        return np.ascontiguousarray(chars[:, :80]), chars[:, 80].astype(np.int32)
    if means is None:
        means = _class_means(wl)
    ncls = CLASSES[wl.model]
    p = rng.dirichlet(np.full(ncls, 0.5))
    y = rng.choice(ncls, size=n, p=p).astype(np.int32)
    x = means[y] + rng.standard_normal((n, FEATURES[wl.model]), dtype=np.float32)
    return x.astype(np.float32), y


def population(wl: Workload, sizes: Optional[np.ndarray] = None, clients=None):
    """Concatenated client-major data for the clients listed (default: all).

    Returns (sizes int64[n_pop], x, y) where x/y hold the listed clients'
    data in client-id order and sizes of unlisted clients are kept (their
    rows are absent).  With clients=None, the full population.
    """
    if sizes is None:
        sizes = client_sizes(wl)
    ids = range(wl.n_pop) if clients is None else sorted(int(c) for c in clients)
    means = None if wl.model == "lstm" else _class_means(wl)
    xs, ys = [], []
    for k in ids:
        x, y = client_data(wl, k, int(sizes[k]), means)
        xs.append(x)
        ys.append(y)
    return sizes, np.concatenate(xs), np.concatenate(ys)


def init_params(model: str, seed: int = MASTER_SEED) -> np.ndarray:
    """theta_g, float32 canonical flat layout."""
    rng = _rng(seed, 3)
    out = []
    for _, shape, init in _param_tensors(model):
        if init[0] == "n":
            out.append(rng.standard_normal(shape).ravel())
        else:
            out.append(rng.uniform(-init[1], init[1], size=shape).ravel())
    return np.concatenate(out).astype(np.float32)


def population_torch(wl: Workload, sizes: np.ndarray, device):
    """Device-side draws for throughput-only runs too large for host numpy.

    Same laws as `population`, different generator (torch Philox): the
    values differ from the numpy path, which is used for every oracle
    comparison.  Returns (x, y) torch tensors, client-major.
    """
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(wl.seed * 7 + 2)
    total = int(sizes.sum())
    ncls = CLASSES[wl.model]
    if wl.model == "lstm":
        p = torch.tensor(_zipf_p(), device=device, dtype=torch.float32)
        chars = torch.multinomial(p, total * 81, replacement=True, generator=g).view(total, 81)
        return chars[:, :80].to(torch.uint8).contiguous(), chars[:, 80].to(torch.int32).contiguous()
    means = torch.from_numpy(_class_means(wl)).to(device)
    rng = _rng(wl.seed, 2, 1 << 30)
    y_np = np.empty(total, dtype=np.int32)
    off = 0
    for k in range(wl.n_pop):
        n = int(sizes[k])
        p = rng.dirichlet(np.full(ncls, 0.5))
        y_np[off:off + n] = rng.choice(ncls, size=n, p=p)
        off += n
    y = torch.from_numpy(y_np).to(device)
    x = torch.empty((total, FEATURES[wl.model]), device=device, dtype=torch.float32)
    chunk = 1 << 16
    for s in range(0, total, chunk):
        e = min(total, s + chunk)
        x[s:e].normal_(generator=g)
        x[s:e] += means[y[s:e].long()]
    return x, y
