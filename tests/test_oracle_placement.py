"""Pins for the oracle's placement, packer and permutation (no GPU).

Placement follows PAPER.md §5 (L358-388); the pins are SPEC.md's hand
traces (tests/golden/spec_examples.json), an exhaustive optimum on tiny
instances with Graham's LPT bound, and invariants (conservation,
determinism, input-order independence).
"""
import itertools
import json
import math
import os

import numpy as np
import pytest

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def lists(ids, off):
    return [list(ids[off[w]:off[w + 1]]) for w in range(len(off) - 1)]


@pytest.mark.parametrize("pol", ["rr", "srr", "bu", "lb"])
def test_spec_worked_examples(pol):
    for ex in GOLD[pol]:
        ids, off = oracle.place(pol, ex["cohort"], ex["sizes"], ex["B"], ex["G"], lb=ex.get("coef"))
        got = lists(ids, off)
        if "expect" in ex:
            assert got == ex["expect"], ex["cite"]
        if "expect_sizes" in ex:
            assert [len(l) for l in got] == ex["expect_sizes"], ex["cite"]
        if "loads" in ex:
            sizes = np.asarray(ex["sizes"])
            assert [int(sizes[l].sum()) for l in got] == ex["loads"], ex["cite"]


def test_eq3_examples():
    for ex in GOLD["eq3"]:
        assert oracle.eq3(ex["coef"], ex["m"]) == pytest.approx(ex["expect"], rel=1e-12), ex["cite"]
    # positivity clamp over [1, 1e5] for a fit with negative terms (reading A23)
    for m in np.geomspace(1, 1e5, 50):
        assert oracle.eq3([0.001, -5.0, 0.5, -1.0], m) > 0


def _brute_opt(costs, G):
    best = math.inf
    for assign in itertools.product(range(G), repeat=len(costs)):
        loads = [0] * G
        for c, w in zip(costs, assign):
            loads[w] += c
        best = min(best, max(loads))
    return best


def test_bu_against_exhaustive_optimum():
    """Greedy LPT: makespan ≤ (4/3 − 1/(3G))·OPT (Graham 1969) and
    max−min load ≤ max m; OPT by brute force, N ≤ 8, G ≤ 3."""
    rng = np.random.default_rng(7)
    for _ in range(120):
        N = int(rng.integers(1, 9))
        G = int(rng.integers(1, 4))
        sizes = rng.integers(1, 60, size=N)
        ids, off = oracle.place("bu", np.arange(N), sizes, 1, G)
        loads = [int(sizes[l].sum()) for l in lists(ids, off)]
        opt = _brute_opt(list(sizes), G)
        assert max(loads) <= (4 / 3 - 1 / (3 * G)) * opt + 1e-9
        assert max(loads) - min(loads) <= sizes.max()
        assert max(loads) <= sizes.sum() / G + sizes.max()


@pytest.mark.parametrize("pol", ["rr", "srr", "bu", "lb"])
def test_conservation_and_determinism(pol):
    rng = np.random.default_rng(3)
    for _ in range(50):
        npop = int(rng.integers(1, 300))
        sizes = rng.integers(1, 3000, size=npop)
        K = int(rng.integers(0, npop + 1))
        cohort = rng.choice(npop, size=K, replace=False)
        G = int(rng.integers(1, 9))
        B = int(rng.integers(1, 64))
        coef = [0.02, 0.5, 1.0, 0.1]
        a = oracle.place(pol, cohort, sizes, B, G, lb=coef)
        b = oracle.place(pol, cohort, sizes, B, G, lb=coef)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
        assert sorted(a[0].tolist()) == sorted(cohort.tolist())
        assert a[1][0] == 0 and a[1][-1] == K and np.all(np.diff(a[1]) >= 0)
        if pol != "rr":  # sorted policies do not depend on cohort input order
            c = oracle.place(pol, rng.permutation(cohort), sizes, B, G, lb=coef)
            assert np.array_equal(a[0], c[0]) and np.array_equal(a[1], c[1])


def test_bu_bootstrap_first_k_one_per_worker():
    """'the first k clients of the list are assigned the same way as the
    previous strategy' — the k largest go one per worker."""
    sizes = np.array([100, 90, 80, 70, 3, 2, 1])
    ids, off = oracle.place("bu", np.arange(7), sizes, 1, 4)
    firsts = [ids[off[w]] for w in range(4)]
    assert firsts == [0, 1, 2, 3]


def test_degenerate_K_equals_G():
    """clients per round = workers → every policy gives one client per worker."""
    sizes = np.array([5, 17, 2, 40, 9, 11, 3, 8, 6, 30])
    for pol in ["rr", "srr", "bu", "lb"]:
        ids, off = oracle.place(pol, np.arange(10), sizes, 4, 10, lb=[1, 0, 1, 0])
        assert np.all(np.diff(off) == 1)


def test_pack_bruteforce():
    rng = np.random.default_rng(11)
    for _ in range(30):
        npop = 50
        sizes = rng.integers(1, 500, size=npop)
        ids = rng.choice(npop, size=20, replace=False)
        B, E = int(rng.integers(1, 40)), int(rng.integers(1, 4))
        seg, steps = oracle.pack(ids, sizes, B, E)
        acc = 0
        for i, c in enumerate(ids):
            assert seg[i] == acc
            acc += sizes[c]
            assert steps[i] == E * -(-sizes[c] // B)
            # m = ceil(n/B) by brute force
            m = 0
            while m * B < sizes[c]:
                m += 1
            assert steps[i] == E * m
        assert seg[-1] == sizes[ids].sum()


def test_splitmix64_reference_vector():
    ex = GOLD["splitmix64"][0]
    gamma = 0x9E3779B97F4A7C15
    got = ["%016x" % oracle.splitmix64((k * gamma) & (2 ** 64 - 1)) for k in range(3)]
    assert got == ex["expect_hex"], ex["cite"]


def test_perm_is_permutation_and_deterministic():
    for n in [0, 1, 2, 7, 100, 2000]:
        p = oracle.perm(230617453, 3, 17, 1, n)
        assert sorted(p.tolist()) == list(range(n))
        assert np.array_equal(p, oracle.perm(230617453, 3, 17, 1, n))
    a = oracle.perm(1, 0, 5, 0, 50)
    b = oracle.perm(1, 0, 5, 1, 50)
    assert not np.array_equal(a, b)  # epochs reshuffle


def test_perm_uniformity():
    """Fisher-Yates with a good mixer: every position of n=4 is uniform over
    4! orderings (chi-square over 24 cells, 24k draws)."""
    counts = {}
    for cid in range(24000):
        p = tuple(oracle.perm(99, 0, cid, 0, 4).tolist())
        counts[p] = counts.get(p, 0) + 1
    assert len(counts) == 24
    chi2 = sum((c - 1000) ** 2 / 1000 for c in counts.values())
    assert chi2 < 60  # df=23, p≈5e-5
