"""Host-side checks of the C-ABI library (no GPU): it loads, exports every symbol
include/fl.h declares, and its host planning (placement, packer) is bit-exact
against the oracle on thousands of random cohorts (SURVEY §8 b, a1, a2)."""
import os
import re

import numpy as np
import pytest

import oracle
import paper_2306_17453_b200 as fl

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = "".join(open(os.path.join(ROOT, "include", f)).read() for f in sorted(os.listdir(os.path.join(ROOT, "include")))
                  if f.endswith(".h"))
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fl_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = fl.lib()
    decl = declared_symbols()
    assert len(decl) >= 20
    for name in decl:
        assert hasattr(L, name), name
    assert sorted(fl.EXPORTS) == decl


def test_abi_version_and_param_counts():
    assert fl.fl_abi_version() == fl.ABI_VERSION == 3
    for m in ["logreg", "cnn", "speech", "lstm"]:
        assert fl.fl_n_params(m) == oracle.n_params(m)
    assert fl.fl_n_params(17) == 0


@pytest.mark.parametrize("policy", ["bu", "lb", "rr", "srr"])
def test_placement_bit_exact_vs_oracle(policy):
    rng = np.random.default_rng({"bu": 1, "lb": 2, "rr": 3, "srr": 4}[policy])
    for trial in range(1500):
        npop = int(rng.integers(1, 400))
        if trial % 3 == 0:  # heavy-tailed sizes like the paper's workloads (Fig. 1)
            sizes = np.clip(np.rint(np.exp(4.9 + 1.03 * rng.standard_normal(npop))), 1, 5000).astype(np.int64)
        else:
            sizes = rng.integers(1, 60, size=npop)
        K = int(rng.integers(0, npop + 1))
        cohort = rng.choice(npop, size=K, replace=False)
        G = int(rng.integers(1, 9))
        B = int(rng.integers(1, 40))
        coef = [float(rng.uniform(0, 0.1)), float(rng.uniform(-1, 2)), float(rng.uniform(0.1, 3)), float(rng.uniform(-1, 1))]
        ids, off = fl.fl_place_plan(policy, cohort, sizes, B, G, coef)
        oids, ooff = oracle.place(policy, cohort, sizes, B, G, lb=coef)
        assert np.array_equal(ids, oids) and np.array_equal(off, ooff), (trial, policy)


def test_pack_bit_exact_vs_oracle():
    rng = np.random.default_rng(12)
    for _ in range(500):
        npop = int(rng.integers(1, 300))
        sizes = rng.integers(1, 3000, size=npop)
        ids = rng.choice(npop, size=int(rng.integers(0, npop + 1)), replace=False)
        B, E = int(rng.integers(1, 64)), int(rng.integers(1, 4))
        seg, steps = fl.fl_pack_plan(ids, sizes, B, E)
        oseg, osteps = oracle.pack(ids, sizes, B, E)
        assert np.array_equal(seg, oseg) and np.array_equal(steps, osteps)


def test_placement_validation():
    sizes = np.array([5, 3, 2, 1])
    with pytest.raises(fl.FLError) as e:
        fl.fl_place_plan("bu", [0, 0], sizes, 1, 2)  # duplicate id
    assert e.value.status == fl.FL_ERR_INVALID
    with pytest.raises(fl.FLError):
        fl.fl_place_plan("bu", [0, 7], sizes, 1, 2)  # unknown id
    with pytest.raises(fl.FLError):
        fl.fl_place_plan("bu", [0, 1], sizes, 1, 0)  # no workers
    with pytest.raises(fl.FLError):
        fl.fl_place_plan("lb", [0, 1], sizes, 1, 2, None)  # LB without a fit
    with pytest.raises(fl.FLError):
        fl.fl_place_plan("bu", [0, 1], np.array([0, 3]), 1, 2)  # empty client
    ids, off = fl.fl_place_plan("bu", [], sizes, 1, 3)
    assert len(ids) == 0 and list(off) == [0, 0, 0, 0]


def test_no_cpu_fallback():
    """Without a CUDA device the compute entry points refuse (FL_ERR_CUDA)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    sizes = np.array([3, 4])
    x = np.zeros((7, 784), np.float32)
    y = np.zeros(7, np.int32)
    with pytest.raises(fl.FLError) as e:
        fl.fl_round_init(fl.Config(model="logreg", batch_size=2, lr=0.1), sizes, x, y,
                         np.zeros(7850, np.float32))
    assert e.value.status == fl.FL_ERR_CUDA


def test_lb_rejects_invalid_coefficients():
    """Eq. 3 needs c > 0 and finite coefficients (log(c·m)); anything else used to
    make every load comparison false and put the whole cohort on worker 0."""
    sizes = np.arange(1, 7, dtype=np.int64) * 10
    for bad in ([1, 1, -1, 0], [1, 1, 0, 0], [np.nan, 1, 1, 0], [1, np.inf, 1, 0]):
        with pytest.raises(fl.FLError) as e:
            fl.fl_place_plan("lb", range(6), sizes, 4, 2, bad)
        assert e.value.status == fl.FL_ERR_INVALID
        with pytest.raises(fl.FLError) as e:
            fl.fl_place_plan("lb_gpu", range(6), sizes, 4, 2, [1, 1, 1, 0] + list(bad))
        assert e.value.status == fl.FL_ERR_INVALID
    ids, off = fl.fl_place_plan("lb", range(6), sizes, 4, 2, [1, 1, 1, 0])
    assert list(off) == [0, 3, 6]
