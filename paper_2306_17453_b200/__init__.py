"""B200-native FedAvg-round engine (Pollen, arXiv 2306.17453) — Python binding.

Argument marshalling only: every step of the round runs in libfl_b200.so
(include/fl.h), whose compute paths are CUDA kernels for sm_100a.  There is no
CPU fallback: a missing library or a missing GPU raises.

Names follow the C-ABI (fl_round_init, fl_place, fl_train_clients,
fl_aggregate, fl_round, ...).  Host arrays are numpy; device arrays are torch
CUDA tensors (only their data pointers cross the boundary).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libfl_b200.so")

FL_OK, FL_ERR_INVALID, FL_ERR_STATE, FL_ERR_OOM, FL_ERR_CUDA, FL_ERR_NCCL, FL_ERR_EMPTY, FL_ERR_UNSUPPORTED = range(8)
STATUS = {0: "FL_OK", 1: "FL_ERR_INVALID", 2: "FL_ERR_STATE", 3: "FL_ERR_OOM", 4: "FL_ERR_CUDA", 5: "FL_ERR_NCCL",
          6: "FL_ERR_EMPTY", 7: "FL_ERR_UNSUPPORTED"}
MODEL = {"logreg": 0, "cnn": 1, "speech": 2, "lstm": 3}
POLICY = {"bu": 0, "lb": 1, "rr": 2, "srr": 3, "lb_gpu": 4}
ABI_VERSION = 3
AGG_MODE = {"nccl": 0, "peer": 1, "unaggregated": 2}
PEER_BLOB_BYTES = 512

# Symbols include/fl.h declares (checked by tests/test_abi.py).
EXPORTS = ["fl_abi_version", "fl_n_params", "fl_place_plan", "fl_pack_plan", "fl_nccl_unique_id", "fl_round_init",
           "fl_place", "fl_train_clients", "fl_aggregate", "fl_aggregate_async", "fl_synchronize", "fl_round", "fl_fedavg_vectors", "fl_get_local_plan",
           "fl_get_client_params", "fl_get_global_params", "fl_set_global_params", "fl_get_stats",
           "fl_set_profiling", "fl_get_kernel_stats", "fl_get_stream", "fl_last_error", "fl_round_destroy", "fl_debug_read",
           "fl_lb_fit", "fl_set_timing_records", "fl_get_client_times", "fl_peer_export", "fl_peer_connect"]


class FLError(RuntimeError):
    def __init__(self, status, msg=""):
        self.status = status
        super().__init__(f"{STATUS.get(status, status)}: {msg}")


class fl_config(C.Structure):
    _fields_ = [("abi_version", C.c_uint32), ("model", C.c_int32), ("batch_size", C.c_int32),
                ("local_epochs", C.c_int32), ("lr", C.c_float), ("shuffle", C.c_int32), ("seed", C.c_uint64),
                ("min_samples", C.c_int64), ("rank", C.c_int32), ("world_size", C.c_int32), ("device", C.c_int32),
                ("nccl_unique_id", C.c_void_p), ("math", C.c_int32), ("stream", C.c_void_p),
                ("sm_count", C.c_int32), ("agg_mode", C.c_int32)]


class fl_population(C.Structure):
    _fields_ = [("n_clients", C.c_int64), ("n_samples", C.c_void_p), ("feature_dim", C.c_int32),
                ("x", C.c_void_p), ("y", C.c_void_p), ("on_device", C.c_int32)]


class fl_round_stats(C.Structure):
    _fields_ = [("round_ms", C.c_double), ("place_ms", C.c_double), ("stage_ms", C.c_double),
                ("train_ms", C.c_double), ("agg_ms", C.c_double), ("allreduce_ms", C.c_double),
                ("client_updates_per_s", C.c_double), ("clients_total", C.c_int64), ("clients_local", C.c_int64),
                ("samples_total", C.c_int64), ("samples_local", C.c_int64), ("steps_local", C.c_int64),
                ("waves", C.c_int64), ("h2d_bytes", C.c_int64), ("kernels", C.c_int64),
                ("train_end_ms", C.c_double), ("round_ms_max", C.c_double), ("train_end_ms_min", C.c_double),
                ("train_end_ms_max", C.c_double), ("timedelta_ms", C.c_double), ("xfer_bytes", C.c_int64),
                ("sm_count", C.c_int32)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class fl_kernel_stats(C.Structure):
    _fields_ = [("name", C.c_char * 32), ("ms", C.c_double), ("launches", C.c_int64), ("flops", C.c_double),
                ("bytes", C.c_double)]


_lib = None


def lib():
    """The loaded libfl_b200.so (built in-tree on first use if absent or stale)."""
    global _lib
    if _lib is None:
        from . import build as _build
        path = _build.build()
        if not os.path.exists(path):
            raise ImportError(f"libfl_b200.so missing at {path}: run python -m paper_2306_17453_b200.build")
        L = C.CDLL(path)
        vp, i64, i32 = C.c_void_p, C.c_int64, C.c_int32
        sig = {
            "fl_abi_version": (C.c_uint32, []),
            "fl_n_params": (i64, [i32]),
            "fl_place_plan": (C.c_int, [i32, vp, i64, vp, i64, i32, i32, vp, vp, vp]),
            "fl_pack_plan": (C.c_int, [vp, i64, vp, i64, i32, i32, vp, vp]),
            "fl_nccl_unique_id": (C.c_int, [vp]),
            "fl_round_init": (C.c_int, [vp, vp, vp, i64, vp]),
            "fl_place": (C.c_int, [vp, vp, i64, i32, vp, vp, vp]),
            "fl_train_clients": (C.c_int, [vp, i32]),
            "fl_aggregate": (C.c_int, [vp, vp, vp]),
            "fl_aggregate_async": (C.c_int, [vp, vp, vp]),
            "fl_synchronize": (C.c_int, [vp]),
            "fl_round": (C.c_int, [vp, vp, i64, i32, vp, i32, vp]),
            "fl_fedavg_vectors": (C.c_int, [vp, vp, vp, i64, i64, vp, vp]),
            "fl_get_local_plan": (C.c_int, [vp, vp, vp, vp, vp]),
            "fl_get_client_params": (C.c_int, [vp, i64, vp]),
            "fl_get_global_params": (C.c_int, [vp, vp]),
            "fl_set_global_params": (C.c_int, [vp, vp]),
            "fl_get_stats": (C.c_int, [vp, vp]),
            "fl_set_profiling": (C.c_int, [vp, i32]),
            "fl_get_kernel_stats": (C.c_int, [vp, i32, vp]),
            "fl_get_stream": (vp, [vp]),
            "fl_last_error": (C.c_char_p, [vp]),
            "fl_round_destroy": (None, [vp]),
            "fl_debug_read": (C.c_int, [vp, C.c_char_p, vp, i64]),
            "fl_lb_fit": (C.c_int, [vp, vp, i64, vp, vp, vp]),
            "fl_set_timing_records": (C.c_int, [vp, i32]),
            "fl_get_client_times": (C.c_int, [vp, vp, vp, vp, vp]),
            "fl_peer_export": (C.c_int, [vp, i64, vp]),
            "fl_peer_connect": (C.c_int, [vp, vp, i32]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _ptr(a):
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()  # torch tensor


def _i64(a):
    return np.ascontiguousarray(a, dtype=np.int64)


def fl_abi_version() -> int:
    return int(lib().fl_abi_version())


def fl_n_params(model) -> int:
    return int(lib().fl_n_params(MODEL.get(model, model)))


def fl_place_plan(policy, cohort, n_samples, batch_size, world_size, lb_coef=None):
    cohort, n_samples = _i64(cohort), _i64(n_samples)
    ids = np.empty(len(cohort), np.int64)
    off = np.empty(world_size + 1, np.int64)
    lb = None if lb_coef is None else np.ascontiguousarray(lb_coef, np.float64)
    rc = lib().fl_place_plan(POLICY.get(policy, policy), _ptr(cohort), len(cohort), _ptr(n_samples), len(n_samples),
                             batch_size, world_size, _ptr(lb), _ptr(ids), _ptr(off))
    if rc != FL_OK:
        raise FLError(rc, "fl_place_plan")
    return ids, off


def fl_pack_plan(ids, n_samples, batch_size, local_epochs):
    ids, n_samples = _i64(ids), _i64(n_samples)
    seg = np.empty(len(ids) + 1, np.int64)
    steps = np.empty(len(ids), np.int64)
    rc = lib().fl_pack_plan(_ptr(ids), len(ids), _ptr(n_samples), len(n_samples), batch_size, local_epochs,
                            _ptr(seg), _ptr(steps))
    if rc != FL_OK:
        raise FLError(rc, "fl_pack_plan")
    return seg, steps


def fl_lb_fit(m, t):
    """Eq. 3 least-squares fit of timing records (include/fl.h): returns (coef[4], kind, mse)."""
    m = np.ascontiguousarray(m, np.float64)
    t = np.ascontiguousarray(t, np.float64)
    if len(m) != len(t):
        raise FLError(FL_ERR_INVALID, "fl_lb_fit: m and t differ in length")
    coef = np.empty(4, np.float64)
    kind, mse = C.c_int32(0), C.c_double(0.0)
    rc = lib().fl_lb_fit(_ptr(m), _ptr(t), len(m), _ptr(coef), C.byref(kind), C.byref(mse))
    if rc != FL_OK:
        raise FLError(rc, "fl_lb_fit")
    return coef, int(kind.value), float(mse.value)


def fl_nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    rc = lib().fl_nccl_unique_id(C.addressof(buf))
    if rc != FL_OK:
        raise FLError(rc, "fl_nccl_unique_id")
    return bytes(buf)


@dataclass
class Config:
    model: str = "cnn"
    batch_size: int = 32
    local_epochs: int = 1
    lr: float = 0.05
    shuffle: int = 0
    seed: int = 230617453
    min_samples: int = 1
    rank: int = 0
    world_size: int = 1
    device: int = 0
    nccl_unique_id: bytes | None = None
    math: int = 0
    stream: int | None = None
    sm_count: int = 0      # green-context SM partition (include/fl.h): 0 whole GPU, s>0 first part, s<0 remainder
    agg_mode: str = "nccl"  # "nccl" | "peer" | "unaggregated" (include/fl.h fl_agg_mode)


class Ctx:
    """Owner of an fl_ctx*.  Keeps every borrowed buffer alive for its lifetime."""

    def __init__(self, cfg: Config, n_samples, x, y, theta_canon, on_device=None):
        L = lib()
        self._keep = []
        self.cfg = cfg
        uid = None
        if cfg.nccl_unique_id is not None:
            uid = (C.c_uint8 * 128).from_buffer_copy(cfg.nccl_unique_id)
            self._keep.append(uid)
        c = fl_config(ABI_VERSION, MODEL[cfg.model], cfg.batch_size, cfg.local_epochs, cfg.lr, cfg.shuffle,
                      cfg.seed & 0xFFFFFFFFFFFFFFFF, cfg.min_samples, cfg.rank, cfg.world_size, cfg.device,
                      C.addressof(uid) if uid is not None else None, cfg.math, cfg.stream, cfg.sm_count,
                      AGG_MODE[cfg.agg_mode])
        n_samples = _i64(n_samples)
        if on_device is None:
            on_device = not isinstance(x, np.ndarray)
        if isinstance(x, np.ndarray):
            x = np.ascontiguousarray(x)
            y = np.ascontiguousarray(y, dtype=np.int32)
        self._keep += [n_samples, x, y]
        feat = int(np.prod(x.shape[1:])) if len(x.shape) > 1 else 1
        pop = fl_population(len(n_samples), _ptr(n_samples), feat, _ptr(x), _ptr(y), int(bool(on_device)))
        theta = np.ascontiguousarray(theta_canon, dtype=np.float32)
        self.P = len(theta)
        h = C.c_void_p()
        rc = L.fl_round_init(C.byref(c), C.byref(pop), _ptr(theta), len(theta), C.byref(h))
        self._h = h
        if rc != FL_OK:
            msg = L.fl_last_error(h).decode() if h.value else ""
            if h.value:
                L.fl_round_destroy(h)
                self._h = C.c_void_p()
            raise FLError(rc, f"fl_round_init: {msg}")

    # --------------------------------------------------------------- helpers
    def _check(self, rc, what):
        if rc != FL_OK:
            raise FLError(rc, f"{what}: {lib().fl_last_error(self._h).decode()}")

    def close(self):
        if self._h and self._h.value:
            lib().fl_round_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stream(self) -> int:
        return int(lib().fl_get_stream(self._h) or 0)

    # --------------------------------------------------------------- ABI calls
    def fl_place(self, cohort, policy="bu", lb_coef=None):
        cohort = _i64(cohort)
        ids = np.empty(len(cohort), np.int64)
        off = np.empty(self.cfg.world_size + 1, np.int64)
        lb = None if lb_coef is None else np.ascontiguousarray(lb_coef, np.float64)
        self._check(lib().fl_place(self._h, _ptr(cohort), len(cohort), POLICY.get(policy, policy), _ptr(lb),
                                   _ptr(ids), _ptr(off)), "fl_place")
        return ids, off

    def fl_train_clients(self, round_index=0):
        self._check(lib().fl_train_clients(self._h, round_index), "fl_train_clients")

    def fl_aggregate(self, want_params=True):
        out = np.empty(self.P, np.float32) if want_params else None
        tot = C.c_int64(0)
        self._check(lib().fl_aggregate(self._h, _ptr(out), C.byref(tot)), "fl_aggregate")
        return out, int(tot.value)

    def fl_aggregate_async(self, out=None):
        """fl_aggregate without waiting: θ_new lands in `out` (page-locked float32[P], e.g.
        torch.empty(P, pin_memory=True)) once fl_synchronize returns."""
        tot = C.c_int64(0)
        p = None if out is None else C.c_void_p(out.data_ptr() if hasattr(out, "data_ptr") else out.ctypes.data)
        if out is not None and (str(out.dtype) not in ("float32", "torch.float32") or len(out) != self.P):
            raise FLError(FL_ERR_INVALID, "fl_aggregate_async: float32[P] output required")
        self._check(lib().fl_aggregate_async(self._h, p, C.byref(tot)), "fl_aggregate_async")
        return int(tot.value)

    def fl_synchronize(self):
        self._check(lib().fl_synchronize(self._h), "fl_synchronize")

    def fl_round(self, cohort, policy="bu", lb_coef=None, round_index=0, stats=True):
        cohort = _i64(cohort)
        lb = None if lb_coef is None else np.ascontiguousarray(lb_coef, np.float64)
        st = fl_round_stats()
        self._check(lib().fl_round(self._h, _ptr(cohort), len(cohort), POLICY.get(policy, policy), _ptr(lb),
                                   round_index, C.byref(st) if stats else None), "fl_round")
        return st.as_dict() if stats else None

    def fl_fedavg_vectors(self, theta_k, n, theta_g, out):
        """theta_k [K,P], theta_g [P], out [P]: torch CUDA float32 tensors; n host ints."""
        n = _i64(n)
        for t in (theta_k, theta_g, out):
            if str(getattr(t, "dtype", "")) != "torch.float32" or not t.is_cuda or not t.is_contiguous():
                raise FLError(FL_ERR_INVALID, "fl_fedavg_vectors: float32 contiguous CUDA tensors required")
        K, P = theta_k.shape
        self._check(lib().fl_fedavg_vectors(self._h, _ptr(theta_k), _ptr(n), K, P, _ptr(theta_g), _ptr(out)),
                    "fl_fedavg_vectors")

    def fl_get_local_plan(self):
        n = C.c_int64(0)
        self._check(lib().fl_get_local_plan(self._h, None, None, None, C.byref(n)), "fl_get_local_plan")
        k = int(n.value)
        ids, seg, steps = np.empty(k, np.int64), np.empty(k + 1, np.int64), np.empty(k, np.int64)
        self._check(lib().fl_get_local_plan(self._h, _ptr(ids), _ptr(seg), _ptr(steps), C.byref(n)),
                    "fl_get_local_plan")
        return ids, seg, steps

    def fl_get_client_params(self, client_id):
        out = np.empty(self.P, np.float32)
        self._check(lib().fl_get_client_params(self._h, int(client_id), _ptr(out)), "fl_get_client_params")
        return out

    def fl_get_global_params(self):
        out = np.empty(self.P, np.float32)
        self._check(lib().fl_get_global_params(self._h, _ptr(out)), "fl_get_global_params")
        return out

    def fl_set_global_params(self, theta):
        theta = np.ascontiguousarray(theta, np.float32)
        self._check(lib().fl_set_global_params(self._h, _ptr(theta)), "fl_set_global_params")

    def fl_debug_read(self, name, shape, dtype=np.float32):
        """Test-only: copy an activation buffer of the last wave (include/fl_debug.h)."""
        out = np.empty(shape, dtype)
        self._check(lib().fl_debug_read(self._h, name.encode(), _ptr(out), out.nbytes), "fl_debug_read")
        return out

    def fl_set_timing_records(self, on=True):
        self._check(lib().fl_set_timing_records(self._h, int(bool(on))), "fl_set_timing_records")

    def fl_get_client_times(self):
        """LB timing records of the last trained round: (ids, m, t_ms), plan order."""
        n = C.c_int64(0)
        self._check(lib().fl_get_client_times(self._h, None, None, None, C.byref(n)), "fl_get_client_times")
        k = int(n.value)
        ids, m, t = np.empty(k, np.int64), np.empty(k, np.int64), np.empty(k, np.float64)
        self._check(lib().fl_get_client_times(self._h, _ptr(ids), _ptr(m), _ptr(t), C.byref(n)),
                    "fl_get_client_times")
        return ids, m, t

    def fl_peer_export(self, max_clients=0) -> bytes:
        """This rank's peer blob (FL_PEER_BLOB_BYTES opaque bytes) for fl_peer_connect."""
        buf = (C.c_uint8 * PEER_BLOB_BYTES)()
        self._check(lib().fl_peer_export(self._h, int(max_clients), C.addressof(buf)), "fl_peer_export")
        return bytes(buf)

    def fl_peer_connect(self, blobs):
        """blobs: every rank's fl_peer_export bytes, in rank order."""
        if len(blobs) != self.cfg.world_size or any(len(b) != PEER_BLOB_BYTES for b in blobs):
            raise FLError(FL_ERR_INVALID, "fl_peer_connect: one blob of PEER_BLOB_BYTES per rank")
        arr = (C.c_uint8 * (PEER_BLOB_BYTES * len(blobs))).from_buffer_copy(b"".join(blobs))
        self._check(lib().fl_peer_connect(self._h, C.addressof(arr), len(blobs)), "fl_peer_connect")

    def fl_get_stats(self):
        st = fl_round_stats()
        self._check(lib().fl_get_stats(self._h, C.byref(st)), "fl_get_stats")
        return st.as_dict()

    def fl_set_profiling(self, on=True):
        self._check(lib().fl_set_profiling(self._h, int(bool(on))), "fl_set_profiling")

    def fl_get_kernel_stats(self):
        """{name: {ms, launches, flops, bytes}} of every kernel class of the last round."""
        out = {}
        k = 0
        while True:
            st = fl_kernel_stats()
            rc = lib().fl_get_kernel_stats(self._h, k, C.byref(st))
            if rc == FL_ERR_INVALID:
                break
            self._check(rc, "fl_get_kernel_stats")
            if st.launches:
                out[st.name.decode()] = {"ms": st.ms, "launches": st.launches, "flops": st.flops, "bytes": st.bytes}
            k += 1
        return out


def fl_round_init(cfg: Config, n_samples, x, y, theta_canon, on_device=None) -> Ctx:
    return Ctx(cfg, n_samples, x, y, theta_canon, on_device)
