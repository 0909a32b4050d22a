"""Pins for the oracle's FedAvg (Eq. 1-2).

SPEC.md worked examples, grouping/permutation invariance between the
plain definition and Eq. 1-2, convexity, the constant-vector
closed form (exact), identical clients == one client.
"""
import json
import os

import numpy as np
import pytest

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def test_fold_examples():
    for ex in GOLD["fold"]:
        th = np.asarray(ex["clients"], dtype=np.float64)
        out = oracle.fedavg_eq12(th, ex["n"], [0, len(ex["n"])])
        assert np.array_equal(out, np.asarray(ex["expect"])), ex["cite"]
        flat, N = oracle.fedavg(th, ex["n"])
        assert N == ex["N"] and np.array_equal(flat, np.asarray(ex["expect"])), ex["cite"]


def test_final_examples():
    for ex in GOLD["final"]:
        th = np.asarray(ex["partials"], dtype=np.float64)
        out, N = oracle.fedavg(th, ex["N"])
        assert np.allclose(out, ex["expect"], rtol=0, atol=0), ex["cite"]
        # a single partial passes through unchanged
        one, _ = oracle.fedavg(th[:1], ex["N"][:1])
        assert np.array_equal(one, th[0])


def test_grouping_and_permutation_invariance():
    """any grouping of clients into workers = flat weighted mean
    within 1e-12 relative; fold order irrelevant."""
    rng = np.random.default_rng(5)
    K, P = 300, 64
    th = rng.standard_normal((K, P))
    n = rng.integers(1, 10_000, size=K)
    flat, _ = oracle.fedavg(th, n)
    for _ in range(30):
        perm = rng.permutation(K)
        G = int(rng.integers(1, 18))
        cuts = np.sort(rng.choice(np.arange(1, K), size=G - 1, replace=False)) if G > 1 else np.array([], int)
        off = np.concatenate([[0], cuts, [K]])
        out = oracle.fedavg_eq12(th[perm], n[perm], off)
        assert np.allclose(out, flat, rtol=1e-12, atol=1e-12)


def test_convexity():
    rng = np.random.default_rng(6)
    th = rng.standard_normal((50, 40))
    n = rng.integers(1, 100, size=50)
    out, _ = oracle.fedavg(th, n)
    assert np.all(out >= th.min(0) - 1e-15) and np.all(out <= th.max(0) + 1e-15)


def test_constant_vectors_exact():
    """Σ n_k v / Σ n_k == v exactly for fp32 v and integer n_k ≤ 2^11 (closed form:
    n_k·v has ≤ 35 significant bits, sums stay < 2^53)."""
    rng = np.random.default_rng(8)
    v = rng.standard_normal(1000).astype(np.float32).astype(np.float64)
    for K in [1, 2, 17, 1000]:
        n = rng.integers(1, 2049, size=K)
        out, N = oracle.fedavg(np.tile(v, (K, 1)), n)
        assert N == n.sum()
        assert np.array_equal(out, v)
        out12 = oracle.fedavg_eq12(np.tile(v, (K, 1)), n, [0, K])
        assert np.allclose(out12, v, rtol=1e-15, atol=0)


def test_identical_clients_equal_single():
    rng = np.random.default_rng(9)
    v = rng.standard_normal(33)
    out, _ = oracle.fedavg(np.tile(v, (7, 1)), rng.integers(1, 50, size=7))
    assert np.allclose(out, v, rtol=1e-15, atol=0)


def test_equal_weights_arithmetic_mean():
    a, b = np.array([[1.0, -2.0, 5.0]]), np.array([[3.0, 4.0, -1.0]])
    out, _ = oracle.fedavg(np.vstack([a, b]), [7, 7])
    assert np.array_equal(out, ((a + b) / 2)[0])


def test_empty_and_invalid():
    with pytest.raises(ValueError):
        oracle.fedavg(np.zeros((1, 3)), [0])


def test_round_metrics_definitions():
    """SPEC L369 / PAPER L411-415, L471-472: duration = max finish,
    timedelta = max − min, throughput = clients / duration."""
    ex = GOLD["metrics"][0]
    f = np.asarray(ex["finish"])
    assert f.max() == ex["duration"]
    assert f.max() - f.min() == ex["timedelta"]
    assert ex["clients"] / f.max() == pytest.approx(ex["throughput"])
