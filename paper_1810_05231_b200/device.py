"""ctypes binding of ``libpdsdp_b200.so`` (the sm_100a C ABI in
``include/pdsdp_b200.h``).

There is no CPU fallback: if the library is missing or no CUDA device is
visible, every entry point raises.  The library owns its device memory; this
module only passes host numpy buffers across the boundary and keeps them
alive for the duration of each call.
"""

from __future__ import annotations

import ctypes as ct
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PDSDP_B200_LIB") or os.path.join(_HERE, "libpdsdp_b200.so")

OUT_LEN = 16
OUT_EPS_P, OUT_EPS_D, OUT_LAMBDA, OUT_FINITE = 0, 1, 2, 3
OUT_PASSES, OUT_MATVECS, OUT_EIGCONV, OUT_EIGRES = 4, 5, 6, 7
OUT_BLOCK = 11
OUT_DONE = 12
OUT_ERR = 13
OUT_DENSE = 8
OUT_DENSE_EXACT = 14
BLOCK_MAX = 64
KMAX = 128

EINVAL, ECUDA, ENOMEM, ERANK = -1, -2, -3, -4

EXPORTED = (
    "pdsdp_batch_create", "pdsdp_batch_destroy", "pdsdp_batch_info", "pdsdp_batch_stream",
    "pdsdp_opnorm_positions", "pdsdp_opnorm_run", "pdsdp_set_alpha", "pdsdp_reset",
    "pdsdp_iterate", "pdsdp_objective", "pdsdp_download_x", "pdsdp_download_y",
    "pdsdp_apply_M", "pdsdp_apply_M_adjoint", "pdsdp_aproj_psd", "pdsdp_strerror",
    "pdsdp_last_error", "pdsdp_version", "pdsdp_set_timing", "pdsdp_kernel_times",
    "pdsdp_debug", "pdsdp_iterate_many", "pdsdp_set_verify_residual",
    "pdsdp_dense_begin", "pdsdp_iterate_dense",
    "pdsdp_slots", "pdsdp_chunk_launch", "pdsdp_chunk_poll", "pdsdp_chunk_collect",
)


class _Problem(ct.Structure):
    _fields_ = [
        ("n", ct.c_int32), ("m", ct.c_int32), ("p", ct.c_int32), ("reserved", ct.c_int32),
        ("C_packed", ct.c_void_p), ("row_ptr", ct.c_void_p), ("row_idx", ct.c_void_p),
        ("row_val", ct.c_void_p), ("b", ct.c_void_p), ("h", ct.c_void_p),
    ]


_lib = None
_lock = threading.Lock()


def load_library(path: str = LIB_PATH):
    """Load the CUDA library; raises RuntimeError (never falls back)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise RuntimeError(
                f"CUDA library {path} is missing; build it with `make` or "
                "`python -c 'import __graft_entry__ as g; g.build()'` (no CPU fallback)")
        lib = ct.CDLL(path)
        P, I32, I64, D = ct.c_void_p, ct.c_int32, ct.c_int64, ct.c_double
        sig = {
            "pdsdp_batch_create": (ct.c_int, [ct.c_int, P, ct.POINTER(P)]),
            "pdsdp_batch_destroy": (ct.c_int, [P]),
            "pdsdp_batch_info": (ct.c_int, [P, ct.c_int, P]),
            "pdsdp_batch_stream": (P, [P]),
            "pdsdp_opnorm_positions": (ct.c_int, [P, ct.c_int, P, P]),
            "pdsdp_opnorm_run": (ct.c_int, [P, ct.c_int, P, ct.c_int, P]),
            "pdsdp_set_alpha": (ct.c_int, [P, ct.c_int, D]),
            "pdsdp_reset": (ct.c_int, [P, ct.c_int, D]),
            "pdsdp_iterate": (ct.c_int, [P, ct.c_int, P, P, P, P, I32, P]),
            "pdsdp_objective": (ct.c_int, [P, ct.c_int, ct.c_int, P]),
            "pdsdp_download_x": (ct.c_int, [P, ct.c_int, ct.c_int, P]),
            "pdsdp_download_y": (ct.c_int, [P, ct.c_int, ct.c_int, P]),
            "pdsdp_apply_M": (ct.c_int, [P, ct.c_int, P, P]),
            "pdsdp_apply_M_adjoint": (ct.c_int, [P, ct.c_int, P, P]),
            "pdsdp_aproj_psd": (ct.c_int, [I32, P, I32, P, P]),
            "pdsdp_strerror": (ct.c_char_p, [ct.c_int]),
            "pdsdp_last_error": (ct.c_char_p, []),
            "pdsdp_version": (ct.c_int, []),
            "pdsdp_set_timing": (ct.c_int, [P, ct.c_int]),
            "pdsdp_kernel_times": (ct.c_int, [P, P]),
            "pdsdp_set_verify_residual": (ct.c_int, [P, ct.c_int]),
            "pdsdp_debug": (ct.c_int, [P, ct.c_int, P]),
            "pdsdp_iterate_many": (ct.c_int, [P, ct.c_int, P, P, P, P, I32, I32, P, P, P, P]),
            "pdsdp_slots": (ct.c_int, [P, P]),
            "pdsdp_chunk_launch": (ct.c_int, [P, I32, I32, I32, I32, I32, I32, I32, D, P]),
            "pdsdp_chunk_poll": (ct.c_int, [P, I32]),
            "pdsdp_chunk_collect": (ct.c_int, [P, I32, I32, I32, P, P]),
            "pdsdp_dense_begin": (ct.c_int, [P, ct.c_int, ct.c_int]),
            "pdsdp_iterate_dense": (ct.c_int, [P, ct.c_int, I32, I32, P]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        del I64
        _lib = lib
        return lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ct.c_void_p) if a is not None else None


def _check(rc: int):
    if rc == 0:
        return
    lib = load_library()
    msg = lib.pdsdp_last_error().decode(errors="replace")
    if rc == EINVAL or rc == ERANK:
        raise ValueError(msg)
    raise RuntimeError(f"pdsdp_b200: {lib.pdsdp_strerror(rc).decode()}: {msg}")


class DeviceBatch:
    """A set of independent SDP instances resident on the current GPU."""

    def __init__(self, problems):
        lib = load_library()
        self._keep = []
        arr = (_Problem * len(problems))()
        for k, prob in enumerate(problems):
            indptr, idx, val = prob.stacked_arrays()
            C = np.ascontiguousarray(prob.C.data, dtype=np.float64)
            indptr = np.ascontiguousarray(indptr, dtype=np.int64)
            idx = np.ascontiguousarray(idx, dtype=np.int64)
            val = np.ascontiguousarray(val, dtype=np.float64)
            b = np.ascontiguousarray(prob.b, dtype=np.float64)
            h = np.ascontiguousarray(prob.h, dtype=np.float64)
            self._keep += [C, indptr, idx, val, b, h]
            arr[k] = _Problem(prob.n, prob.m, prob.p, 0, C.ctypes.data, indptr.ctypes.data,
                              idx.ctypes.data, val.ctypes.data, b.ctypes.data, h.ctypes.data)
        handle = ct.c_void_p()
        _check(lib.pdsdp_batch_create(len(problems), ct.cast(arr, ct.c_void_p), ct.byref(handle)))
        self._keep = []
        self.h = handle
        self.lib = lib
        self.problems = list(problems)
        self.count = len(problems)

    def close(self):
        if getattr(self, "h", None):
            self.lib.pdsdp_batch_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self, inst: int = 0) -> dict:
        out = np.zeros(8, dtype=np.int64)
        _check(self.lib.pdsdp_batch_info(self.h, inst, _ptr(out)))
        keys = ("n", "z_slots", "t_space", "cluster", "ld", "group", "smem", "device_bytes")
        return dict(zip(keys, out.tolist()))

    def stream_handle(self) -> int:
        return self.lib.pdsdp_batch_stream(self.h) or 0

    def set_timing(self, enable: bool):
        _check(self.lib.pdsdp_set_timing(self.h, 1 if enable else 0))

    def set_verify_residual(self, enable: bool):
        """Also evaluate ||dX/alpha||_F^2 entry by entry after each step
        (output slot OUT_DENSE_EXACT) next to the factored form (OUT_DENSE)."""
        _check(self.lib.pdsdp_set_verify_residual(self.h, 1 if enable else 0))

    def kernel_times(self) -> dict:
        out = np.zeros(5)
        _check(self.lib.pdsdp_kernel_times(self.h, _ptr(out)))
        return {"iterate_ms": out[0], "iterations": int(out[1]),
                "residual_ms": out[2], "residual_launches": int(out[3]), "launches": int(out[4])}

    def debug(self, inst: int = 0) -> dict:
        out = np.zeros(4504 + 16 * 2048)
        _check(self.lib.pdsdp_debug(self.h, inst, _ptr(out)))
        bh = int(out[400 + 4096])
        return {"passes": out[:256].reshape(32, 8), "theta": out[256:320], "res": out[320:384],
                "prof_cycles": out[384:400], "raw": out,
                "H": out[400:400 + bh * bh].reshape(bh, bh) if bh > 0 else None}

    # ---- operator norm (problem.py:157-185) ----
    def opnorm_positions(self, inst: int) -> np.ndarray:
        cnt = ct.c_int64()
        _check(self.lib.pdsdp_opnorm_positions(self.h, inst, None, ct.byref(cnt)))
        pos = np.zeros(cnt.value, dtype=np.int64)
        _check(self.lib.pdsdp_opnorm_positions(self.h, inst, _ptr(pos), ct.byref(cnt)))
        return pos

    def opnorm_run(self, inst: int, x0, iters: int) -> np.ndarray:
        s = np.zeros(iters)
        x0p = None
        if x0 is not None:
            x0 = np.ascontiguousarray(x0, dtype=np.float64)
            x0p = _ptr(x0)
        _check(self.lib.pdsdp_opnorm_run(self.h, inst, x0p, iters, _ptr(s)))
        return s

    def set_alpha(self, inst: int, alpha: float):
        _check(self.lib.pdsdp_set_alpha(self.h, inst, float(alpha)))

    def reset(self, inst: int, seed: float = 0.0):
        _check(self.lib.pdsdp_reset(self.h, inst, float(seed)))

    def iterate(self, insts, ranks, ypars, flags=None, maxpass: int = 60) -> np.ndarray:
        insts = np.ascontiguousarray(insts, dtype=np.int32)
        ranks = np.ascontiguousarray(ranks, dtype=np.int32)
        ypars = np.ascontiguousarray(ypars, dtype=np.int32)
        fl = None if flags is None else np.ascontiguousarray(flags, dtype=np.int32)
        out = np.zeros((insts.size, OUT_LEN))
        _check(self.lib.pdsdp_iterate(self.h, insts.size, _ptr(insts), _ptr(ranks), _ptr(ypars),
                                      _ptr(fl), int(maxpass), _ptr(out)))
        return out

    def iterate_many(self, insts, ranks, ypar0, K: int, conv_thr, stall_thr, flags=None,
                     maxpass: int = 60):
        """Up to K steps per instance; returns (out[nact, K, OUT_LEN], steps_done[nact])."""
        insts = np.ascontiguousarray(insts, dtype=np.int32)
        ranks = np.ascontiguousarray(ranks, dtype=np.int32)
        ypar0 = np.ascontiguousarray(ypar0, dtype=np.int32)
        fl = None if flags is None else np.ascontiguousarray(flags, dtype=np.int32)
        conv = np.ascontiguousarray(conv_thr, dtype=np.float64)
        stall = np.ascontiguousarray(stall_thr, dtype=np.float64).reshape(insts.size, K)
        out = np.zeros((insts.size, K, OUT_LEN))
        done = np.zeros(insts.size, dtype=np.int32)
        _check(self.lib.pdsdp_iterate_many(self.h, insts.size, _ptr(insts), _ptr(ranks), _ptr(ypar0),
                                           _ptr(fl), int(maxpass), int(K), _ptr(conv), _ptr(stall),
                                           _ptr(out), _ptr(done)))
        return out, done

    # ---- asynchronous per-instance chunks (one stream per resident cluster) ----
    def slots(self) -> int:
        n = ct.c_int32()
        _check(self.lib.pdsdp_slots(self.h, ct.byref(n)))
        return int(n.value)

    def chunk_launch(self, slot: int, inst: int, rank: int, ypar0: int, K: int, conv_thr: float,
                     stall_thr, flags: int = 0, maxpass: int = 60):
        stall = np.ascontiguousarray(stall_thr, dtype=np.float64)
        assert stall.size == K
        _check(self.lib.pdsdp_chunk_launch(self.h, slot, inst, int(rank), int(ypar0), int(flags),
                                           int(maxpass), int(K), float(conv_thr), _ptr(stall)))

    def chunk_poll(self, slot: int) -> bool:
        rc = self.lib.pdsdp_chunk_poll(self.h, slot)
        if rc < 0:
            _check(rc)
        return rc == 1

    def chunk_collect(self, slot: int, inst: int, K: int):
        out = np.zeros((K, OUT_LEN))
        done = ct.c_int32()
        _check(self.lib.pdsdp_chunk_collect(self.h, slot, inst, int(K), _ptr(out), ct.byref(done)))
        return out, int(done.value)

    def dense_begin(self, inst: int, from_factored: bool):
        """Switch an instance to the dense-iterate path (full device
        eigendecomposition): X_k expanded from its factors, or X_0 = 0."""
        _check(self.lib.pdsdp_dense_begin(self.h, inst, 1 if from_factored else 0))

    def iterate_dense(self, inst: int, r: int, ypar: int) -> np.ndarray:
        out = np.zeros(OUT_LEN)
        _check(self.lib.pdsdp_iterate_dense(self.h, inst, int(r), int(ypar), _ptr(out)))
        return out

    def objective(self, inst: int, which: int = 0) -> float:
        v = np.zeros(1)
        _check(self.lib.pdsdp_objective(self.h, inst, which, _ptr(v)))
        return float(v[0])

    def download_x(self, inst: int, which: int = 0) -> np.ndarray:
        n = self.problems[inst].n
        out = np.empty(n * (n + 1) // 2)
        _check(self.lib.pdsdp_download_x(self.h, inst, which, _ptr(out)))
        return out

    def download_y(self, inst: int, ypar: int) -> np.ndarray:
        prob = self.problems[inst]
        out = np.zeros(prob.m + prob.p)
        if out.size:
            _check(self.lib.pdsdp_download_y(self.h, inst, ypar, _ptr(out)))
        return out

    def apply_M(self, inst: int, X_packed) -> np.ndarray:
        prob = self.problems[inst]
        X = np.ascontiguousarray(X_packed, dtype=np.float64)
        out = np.zeros(prob.m + prob.p)
        _check(self.lib.pdsdp_apply_M(self.h, inst, _ptr(X), _ptr(out)))
        return out

    def apply_M_adjoint(self, inst: int, y) -> np.ndarray:
        prob = self.problems[inst]
        y = np.ascontiguousarray(y, dtype=np.float64)
        out = np.zeros(prob.packed_len)
        _check(self.lib.pdsdp_apply_M_adjoint(self.h, inst, _ptr(y), _ptr(out)))
        return out


def aproj_psd_packed(n: int, S_packed, r: int):
    lib = load_library()
    S = np.ascontiguousarray(S_packed, dtype=np.float64)
    out = np.zeros(n * (n + 1) // 2)
    lam = ct.c_double()
    _check(lib.pdsdp_aproj_psd(n, _ptr(S), r, _ptr(out), ct.byref(lam)))
    return out, lam.value
