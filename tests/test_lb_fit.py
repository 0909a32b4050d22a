"""LB loop: Eq. 3 fit and per-GPU LB placement.

Oracle pins (no GPU): SPEC's hand trace of per-GPU LB, reduction to the
single-fit LB when all fits are equal, the fit's self-consistency on
noiseless Eq. 3 data and on linear data, least-squares
optimality against random perturbations and against numpy's lstsq on the
reparametrised basis (x, log x, 1), the held-out error on noisy data, and
the positivity / fallback rule.  Then the library (host-only entry
points, no GPU needed) against the oracle: the fit's predictions and the
per-GPU plan bit for bit.  GPU: timing records of a trained round and a 3-round
LB loop through the driver.
"""
import numpy as np
import pytest

import oracle
import synth

GOLD_MODEL = (0.05, 2.0, 0.5, 1.0)


def eq3(coef, m):
    a, b, c, d = coef
    return a * m + b * np.log(c * m) + d


def lists(ids, off):
    return [list(ids[off[w]:off[w + 1]]) for w in range(len(off) - 1)]


# ----------------------------------------------------------------- placement pins
def test_lb_gpu_spec_hand_trace():
    """fits A: t = m, B: t = 2m, batches [4,3,2,1] -> A: [4,2,1], B: [3]."""
    sizes = [4, 3, 2, 1]
    fitA, fitB = [1, 0, 1, 0], [2, 0, 1, 0]
    ids, off = oracle.place_lb_gpu([0, 1, 2, 3], sizes, 1, 2, [fitA, fitB])
    assert lists(ids, off) == [[0, 2, 3], [1]]
    # worker 0 slower: the fastest worker (1) is considered first and takes ties
    ids, off = oracle.place_lb_gpu([0, 1, 2, 3], sizes, 1, 2, [fitB, fitA])
    assert lists(ids, off) == [[1], [0, 2, 3]]


def test_lb_gpu_equal_fits_is_single_fit_lb():
    rng = np.random.default_rng(3)
    for _ in range(30):
        n = rng.integers(1, 400, size=60)
        G = int(rng.integers(1, 6))
        coef = [rng.uniform(0.01, 2), rng.uniform(-1, 1), 1.0, rng.uniform(1, 5)]
        cohort = rng.choice(60, size=int(rng.integers(1, 60)), replace=False)
        a = oracle.place_lb_gpu(cohort, n, 8, G, [coef] * G)
        b = oracle.place("lb", cohort, n, 8, G, lb=coef)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_lb_gpu_conservation_and_faster_worker_gets_more():
    rng = np.random.default_rng(4)
    n = rng.integers(10, 2000, size=300)
    ids, off = oracle.place_lb_gpu(np.arange(300), n, 32, 2, [[1, 0, 1, 0.5], [3, 0, 1, 1.5]])
    assert sorted(ids.tolist()) == list(range(300))
    mA = np.ceil(n[ids[off[0]:off[1]]] / 32).sum()
    mB = np.ceil(n[ids[off[1]:off[2]]] / 32).sum()
    assert mA > 2.5 * mB  # a 3x faster GPU receives ~3x the batches


# ----------------------------------------------------------------- fit pins
def test_fit_noiseless_eq3_data():
    """predictions match the generator within 1e-3 (here 1e-9: the data are exact).
    S:228 samples m in [1, 500], but its generator predicts t(1) = 0.05 + 2·log 0.5 + 1 < 0,
    which no accepted (positive) fit can reproduce: m starts at 2 here."""
    m = np.linspace(2, 500, 100)
    t = eq3(GOLD_MODEL, m)
    coef, kind, mse = oracle.eq3_fit(m, t)
    assert kind == 0 and coef[2] == 1.0
    assert np.max(np.abs(eq3(coef, m) / t - 1)) < 1e-9
    assert mse < 1e-18 * np.mean(t ** 2)
    # b is identifiable, (c, d) only through b·log c + d
    assert coef[0] == pytest.approx(0.05, rel=1e-9) and coef[1] == pytest.approx(2.0, rel=1e-9)
    assert coef[3] == pytest.approx(2.0 * np.log(0.5) + 1.0, rel=1e-9)


def test_fit_linear_data():
    """y = 2m -> predictions within 1% (here exact to rounding)."""
    m = np.arange(1, 101, dtype=float)
    coef, kind, _ = oracle.eq3_fit(m, 2 * m)
    assert np.max(np.abs(eq3(coef, m) - 2 * m)) < 1e-9


def test_fit_is_least_squares_minimum():
    rng = np.random.default_rng(5)
    m = rng.integers(1, 800, size=200).astype(float)
    t = eq3((0.02, 3.0, 1.0, 4.0), m) * (1 + 0.1 * rng.standard_normal(200))
    coef, kind, mse = oracle.eq3_fit(m, t)
    assert kind == 0
    # numpy's least squares over the reparametrised basis (x, log x, 1) — a library witness
    X = np.stack([m, np.log(m), np.ones_like(m)], 1)
    beta = np.linalg.lstsq(X, t, rcond=None)[0]
    assert np.allclose([coef[0], coef[1], coef[3]], beta, rtol=1e-7, atol=1e-9)
    # no nearby (a, b, c, d) — including other c — does better
    for _ in range(300):
        pert = np.array(coef) * (1 + 1e-3 * rng.standard_normal(4))
        assert np.mean((eq3(pert, m) - t) ** 2) >= mse * (1 - 1e-12)
    for c in (0.1, 0.5, 2.0, 10.0):  # c only shifts d: the minimum over (a, b, d) is the same
        Xc = np.stack([m, np.log(c * m), np.ones_like(m)], 1)
        bc = np.linalg.lstsq(Xc, t, rcond=None)[0]
        assert np.mean((Xc @ bc - t) ** 2) == pytest.approx(mse, rel=1e-9)


def test_fit_noisy_heldout():
    """1 % relative noise, 500 points -> held-out MSE <= 2x the noise floor."""
    rng = np.random.default_rng(6)
    m = rng.integers(2, 500, size=1000).astype(float)
    clean = eq3(GOLD_MODEL, m)
    t = clean * (1 + 0.01 * rng.standard_normal(1000))
    coef, kind, _ = oracle.eq3_fit(m[:500], t[:500])
    floor = np.mean((t[500:] - clean[500:]) ** 2)
    assert np.mean((eq3(coef, m[500:]) - t[500:]) ** 2) <= 2 * floor


def test_fit_positivity_fallback():
    """an accepted fit has a >= 0 and is positive on the observed range."""
    m = np.arange(1, 41, dtype=float)
    # decreasing times: Eq. 3's LS fit has a < 0 -> the line also has a < 0 -> constant
    coef, kind, _ = oracle.eq3_fit(m, 100.0 - m)
    assert kind == 2 and coef[0] == 0 and coef[3] == pytest.approx(np.mean(100.0 - m))
    # a log-shaped cloud that dips below zero at small m: Eq. 3 rejected, line accepted
    t = 10 * np.log(m) - 5 + 0.01 * m
    coef, kind, _ = oracle.eq3_fit(m, t)
    assert kind == 1 and coef[0] >= 0
    assert np.all(eq3(coef, m) > 0)
    with pytest.raises(ValueError):
        oracle.eq3_fit([1, 2, 3], [1, 2, 3])  # < 4 records


# ----------------------------------------------------------------- library vs oracle (host-only)
def test_library_fit_matches_oracle():
    fl = pytest.importorskip("paper_2306_17453_b200")
    rng = np.random.default_rng(8)
    for trial in range(40):
        n = int(rng.integers(4, 300))
        m = rng.integers(1, int(rng.integers(2, 2000)), size=n).astype(float)
        gen = (rng.uniform(0, 1), rng.uniform(-3, 3), rng.uniform(0.2, 5), rng.uniform(0, 10))
        t = eq3(gen, m) + rng.uniform(0, 2) * rng.standard_normal(n)
        c1, k1, e1 = fl.fl_lb_fit(m, t)
        c0, k0, e0 = oracle.eq3_fit(m, t)
        assert k1 == k0, trial
        assert np.allclose(eq3(c1, m), eq3(c0, m), rtol=1e-7, atol=1e-9 * np.max(np.abs(t))), trial
        assert e1 == pytest.approx(e0, rel=1e-6, abs=1e-12)
    with pytest.raises(fl.FLError):
        fl.fl_lb_fit([1, 2, 3], [1, 2, 3])
    with pytest.raises(fl.FLError):  # non-finite records are rejected, not fitted
        fl.fl_lb_fit([1, 2, 3, 4], [1.0, np.nan, 3.0, 4.0])
    with pytest.raises(fl.FLError):
        fl.fl_lb_fit([1, 2, np.inf, 4], [1.0, 2.0, 3.0, 4.0])


def test_library_lb_gpu_plan_bit_exact():
    fl = pytest.importorskip("paper_2306_17453_b200")
    rng = np.random.default_rng(9)
    sizes = synth.client_sizes(synth.preset("C3"))
    for trial in range(25):
        G = int(rng.integers(1, 9))
        cohort = rng.choice(len(sizes), size=int(rng.integers(0, 1000)), replace=False)
        coef = np.stack([rng.uniform(0.01, 3, G), rng.uniform(-2, 2, G), rng.uniform(0.5, 2, G),
                         rng.uniform(0.1, 5, G)], 1)
        a = fl.fl_place_plan("lb_gpu", cohort, sizes, 32, G, coef)
        b = oracle.place_lb_gpu(cohort, sizes, 32, G, coef)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]), trial


# ----------------------------------------------------------------- GPU
def _ctx(model, wl_name, **kw):
    import paper_2306_17453_b200 as fl
    wl = synth.preset(wl_name, **kw)
    sizes = synth.client_sizes(wl)
    _, x, y = synth.population(wl, sizes)
    theta = synth.init_params(model)
    cfg = fl.Config(model=model, batch_size=wl.B, local_epochs=wl.E, lr=wl.lr)
    return fl.fl_round_init(cfg, sizes, x, y, theta), sizes, wl


@pytest.mark.gpu
def test_timing_records_cnn():
    import paper_2306_17453_b200 as fl
    ctx, sizes, wl = _ctx("cnn", "C2", n_pop=24, n_cohort=24)
    with pytest.raises(fl.FLError):
        ctx.fl_get_client_times()  # no round with records yet
    ctx.fl_set_timing_records(True)
    st = ctx.fl_round(np.arange(24), policy="bu")
    ids, m, t = ctx.fl_get_client_times()
    pids, _, _ = ctx.fl_get_local_plan()
    assert np.array_equal(ids, pids)
    assert np.array_equal(m, (sizes[ids] + wl.B - 1) // wl.B)
    assert np.all(t > 0) and np.all(t <= st["train_ms"] * 1.001 + 0.01)
    # the last client to finish ends the training phase; bigger clients finish later
    assert t.max() == pytest.approx(st["train_ms"], rel=0.05)
    assert np.corrcoef(m, t)[0, 1] > 0.5
    coef, kind, _ = fl.fl_lb_fit(m, t)
    assert kind in (0, 1, 2)


@pytest.mark.gpu
def test_lb_loop_three_rounds():
    """RR bootstrap, then per-GPU Eq. 3 fits drive the placement."""
    from paper_2306_17453_b200.driver import RoundDriver, sample_cohort
    import paper_2306_17453_b200 as fl
    ctx, sizes, wl = _ctx("cnn", "C2", n_pop=40, n_cohort=40)
    drv = RoundDriver(ctx, policy="lb")
    for r in range(3):
        cohort = sample_cohort(40, 16, seed=1, round_index=r)
        st = drv.run(cohort, r)
        assert st["clients_total"] == 16
    assert [h[0] for h in drv.history] == ["rr", "lb_gpu", "lb_gpu"]
    assert drv.coef.shape == (1, 4) and np.all(np.isfinite(drv.coef))
    theta = ctx.fl_get_global_params()
    assert np.all(np.isfinite(theta))
    # records accumulate across rounds ("keep all the data")
    assert sum(len(r[0]) for r in drv.records) == 48


@pytest.mark.gpu
def test_timing_records_logreg_and_lstm():
    """Every model records: logreg trains all clients in one launch (one shared record),
    the LSTM's waves are serial, so a client with more steps finishes strictly later."""
    import paper_2306_17453_b200 as fl
    ctx, sizes, wl = _ctx("logreg", "C1")
    ctx.fl_set_timing_records(True)
    ctx.fl_round(synth.cohort(wl))
    ids, m, t = ctx.fl_get_client_times()
    assert len(ids) == wl.n_cohort and np.all(t > 0) and np.all(t == t[0])
    ctx.close()
    wl = synth.preset("C5", n_pop=6, n_cohort=6)
    sizes = np.array([4, 8, 12, 4, 20, 9], dtype=np.int64)
    _, x, y = synth.population(wl, sizes)
    ctx = fl.fl_round_init(fl.Config(model="lstm", batch_size=4, lr=wl.lr), sizes, x, y, synth.init_params("lstm"))
    ctx.fl_set_timing_records(True)
    ctx.fl_round(np.arange(6))
    ids, m, t = ctx.fl_get_client_times()
    for i in range(6):
        for j in range(6):
            if m[i] > m[j]:
                assert t[i] > t[j]
            elif m[i] == m[j]:
                assert t[i] == t[j]
