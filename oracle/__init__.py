"""ctypes binding of the CPU fp64 oracle (oracle/fl_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference leg.  The product package
(paper_2306_17453_b200) never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "fl_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

MODEL = {"logreg": 0, "cnn": 1, "speech": 2, "lstm": 3}
POLICY = {"bu": 0, "lb": 1, "rr": 2, "srr": 3}

_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fPIC", "-shared",
                               "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(build())
        L.orc_splitmix64.restype = C.c_uint64
        L.orc_splitmix64.argtypes = [C.c_uint64]
        L.orc_perm.restype = None
        L.orc_perm.argtypes = [C.c_uint64] * 4 + [C.c_int64, _i64p]
        L.orc_eq3.restype = C.c_double
        L.orc_eq3.argtypes = [_f64p, C.c_double]
        L.orc_place.restype = C.c_int
        L.orc_place.argtypes = [C.c_int, _i64p, C.c_int64, _i64p, C.c_int64, C.c_int64, C.c_int64,
                                C.c_void_p, _i64p, _i64p]
        L.orc_pack.restype = None
        L.orc_pack.argtypes = [_i64p, C.c_int64, _i64p, C.c_int64, C.c_int64, _i64p, _i64p]
        L.orc_n_params.restype = C.c_int64
        L.orc_n_params.argtypes = [C.c_int]
        L.orc_feature_dim.restype = C.c_int
        L.orc_feature_dim.argtypes = [C.c_int]
        L.orc_sample_grad.restype = C.c_double
        L.orc_sample_grad.argtypes = [C.c_int, _f64p, C.c_void_p, C.c_int, _f64p]
        L.orc_local_sgd.restype = C.c_double
        L.orc_local_sgd.argtypes = [C.c_int, _f64p, C.c_int64, C.c_void_p, _i32p, C.c_int64, C.c_int64,
                                    C.c_int64, C.c_double, C.c_int, C.c_uint64, C.c_uint64, C.c_uint64]
        L.orc_train_clients.restype = C.c_int
        L.orc_train_clients.argtypes = [C.c_int, _f64p, C.c_int64, C.c_void_p, _i32p, _i64p, _i64p, C.c_int64,
                                        C.c_int64, C.c_int64, C.c_double, C.c_int, C.c_uint64, C.c_uint64,
                                        _f64p, C.c_int]
        L.orc_fedavg.restype = C.c_int
        L.orc_fedavg.argtypes = [_f64p, _i64p, C.c_int64, C.c_int64, _f64p, C.POINTER(C.c_int64)]
        L.orc_fedavg_eq12.restype = C.c_int
        L.orc_fedavg_eq12.argtypes = [_f64p, _i64p, C.c_int64, C.c_int64, _i64p, C.c_int64, _f64p]
        L.orc_place_lb_gpu.restype = C.c_int
        L.orc_place_lb_gpu.argtypes = [_i64p, C.c_int64, _i64p, C.c_int64, C.c_int64, C.c_int64, C.c_void_p,
                                       _i64p, _i64p]
        L.orc_eq3_fit.restype = C.c_int
        L.orc_eq3_fit.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.POINTER(C.c_double)]
        _lib = L
    return _lib


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


# ------------------------------------------------------------------ API
def splitmix64(x: int) -> int:
    return int(lib().orc_splitmix64(x & 0xFFFFFFFFFFFFFFFF))


def perm(seed: int, rnd: int, cid: int, epoch: int, n: int) -> np.ndarray:
    out = np.empty(n, dtype=np.int64)
    lib().orc_perm(seed, rnd, cid, epoch, n, out)
    return out


def eq3(coef, m: float) -> float:
    return float(lib().orc_eq3(np.ascontiguousarray(coef, dtype=np.float64), float(m)))


def place(policy: str, cohort, n_samples, B: int, G: int, lb=None):
    """Returns (ids[K], off[G+1]) — per-worker lists in assignment order."""
    cohort = _i64(cohort)
    n_samples = _i64(n_samples)
    ids = np.empty(len(cohort), dtype=np.int64)
    off = np.empty(G + 1, dtype=np.int64)
    lbp = None
    if lb is not None:
        lbarr = np.ascontiguousarray(lb, dtype=np.float64)
        lbp = lbarr.ctypes.data
    rc = lib().orc_place(POLICY[policy], cohort, len(cohort), n_samples, len(n_samples), B, G, lbp, ids, off)
    if rc != 0:
        raise ValueError("invalid placement input")
    return ids, off


def place_lb_gpu(cohort, n_samples, B: int, G: int, coef):
    """LB with one Eq. 3 fit per worker, coef [G][4]. Returns (ids[K], off[G+1])."""
    cohort, n_samples = _i64(cohort), _i64(n_samples)
    coef = np.ascontiguousarray(coef, dtype=np.float64).reshape(G, 4)
    ids = np.empty(len(cohort), dtype=np.int64)
    off = np.empty(G + 1, dtype=np.int64)
    rc = lib().orc_place_lb_gpu(cohort, len(cohort), n_samples, len(n_samples), B, G, coef.ctypes.data, ids, off)
    if rc != 0:
        raise ValueError("invalid placement input")
    return ids, off


def eq3_fit(m, t):
    """Least-squares Eq. 3 fit: (coef[4], kind, mse); kind 0 Eq. 3, 1 line, 2 constant."""
    m = np.ascontiguousarray(m, dtype=np.float64)
    t = np.ascontiguousarray(t, dtype=np.float64)
    coef = np.empty(4, dtype=np.float64)
    mse = C.c_double(0.0)
    kind = lib().orc_eq3_fit(m.ctypes.data, t.ctypes.data, len(m), coef.ctypes.data, C.byref(mse))
    if kind < 0:
        raise ValueError("eq3_fit needs >= 4 records with m >= 1")
    return coef, int(kind), float(mse.value)


def pack(ids, n_samples, B: int, E: int):
    ids = _i64(ids)
    seg = np.empty(len(ids) + 1, dtype=np.int64)
    steps = np.empty(len(ids), dtype=np.int64)
    lib().orc_pack(ids, len(ids), _i64(n_samples), B, E, seg, steps)
    return seg, steps


def n_params(model: str) -> int:
    return int(lib().orc_n_params(MODEL[model]))


def feature_dim(model: str) -> int:
    return int(lib().orc_feature_dim(MODEL[model]))


def _xarr(model, x):
    return np.ascontiguousarray(x, dtype=np.uint8 if model == "lstm" else np.float32)


def sample_grad(model: str, theta, x, y: int):
    th = np.ascontiguousarray(theta, dtype=np.float64)
    g = np.empty(n_params(model), dtype=np.float64)
    xa = _xarr(model, x)
    loss = lib().orc_sample_grad(MODEL[model], th, xa.ctypes.data, int(y), g)
    return loss, g


def local_sgd(model: str, theta_g, x, y, B: int, E: int, lr: float, shuffle=0, seed=0, rnd=0, cid=0):
    """One client's ClientUpdate; returns fp64 θ_k."""
    th = np.array(theta_g, dtype=np.float64, copy=True)
    xa = _xarr(model, x)
    ya = np.ascontiguousarray(y, dtype=np.int32)
    lib().orc_local_sgd(MODEL[model], th, th.size, xa.ctypes.data, ya, len(ya), B, E, lr, shuffle, seed, rnd, cid)
    return th


def train_clients(model: str, theta_g, x, y, pop_off, ids, B, E, lr, shuffle=0, seed=0, rnd=0, threads=0):
    """fp64 θ_k for each id (in the given order) and the thread count used."""
    th = np.ascontiguousarray(theta_g, dtype=np.float64)
    ids = _i64(ids)
    out = np.empty((len(ids), th.size), dtype=np.float64)
    xa = _xarr(model, x)
    used = lib().orc_train_clients(MODEL[model], th, th.size, xa.ctypes.data, np.ascontiguousarray(y, dtype=np.int32),
                                   _i64(pop_off), ids, len(ids), B, E, lr, shuffle, seed, rnd, out, threads)
    return out, used


def fedavg(theta_k, n):
    """Plain definition Σ n_k θ_k / Σ n_k in fp64 → (θ, N)."""
    tk = np.ascontiguousarray(theta_k, dtype=np.float64)
    K, P = tk.shape
    out = np.empty(P, dtype=np.float64)
    tot = C.c_int64(0)
    rc = lib().orc_fedavg(tk, _i64(n), K, P, out, C.byref(tot))
    if rc != 0:
        raise ValueError("fedavg: empty or invalid weights")
    return out, int(tot.value)


def fedavg_eq12(theta_k, n, worker_off):
    tk = np.ascontiguousarray(theta_k, dtype=np.float64)
    K, P = tk.shape
    out = np.empty(P, dtype=np.float64)
    off = _i64(worker_off)
    rc = lib().orc_fedavg_eq12(tk, _i64(n), K, P, off, len(off) - 1, out)
    if rc != 0:
        raise ValueError("fedavg_eq12: empty")
    return out


def fedavg_round(model, theta_g, x, y, sizes, cohort, B, E, lr, shuffle=0, seed=0, rnd=0, threads=0, pop_ids=None):
    """The whole round by its plain definition: every cohort client's local SGD
    from θ_g, then the sample-weighted mean.  x/y hold the data of `pop_ids`
    (default: every population client) client-major.  Returns (θ_new fp64, N, θ_k)."""
    sizes = _i64(sizes)
    if pop_ids is None:
        pop_off = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    else:
        # offsets for a partial population: clients not in pop_ids get zero-length rows
        present = np.zeros(len(sizes), dtype=np.int64)
        present[np.asarray(sorted(pop_ids))] = sizes[np.asarray(sorted(pop_ids))]
        pop_off = np.concatenate([[0], np.cumsum(present)]).astype(np.int64)
    tk, _ = train_clients(model, theta_g, x, y, pop_off, cohort, B, E, lr, shuffle, seed, rnd, threads)
    out, N = fedavg(tk, sizes[_i64(cohort)])
    return out, N, tk
