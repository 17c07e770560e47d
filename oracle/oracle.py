"""ctypes front-end of oracle/qgemm_oracle.c (TEST INFRASTRUCTURE ONLY).

Arrays use the storage convention of the paper's column-major, interleaved
layout: a numpy float64 array of shape (ncols, ld, 4),
C-contiguous, is exactly column-major storage with leading dimension ``ld``
counted in quaternions and components [q0, q1, q2, q3] contiguous.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "qgemm_oracle.c")
_SO = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

CFLAGS = ["-O3", "-fno-fast-math", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared", "-std=c11"]


def lib_path() -> str:
    return _SO


def build_oracle(force: bool = False) -> str:
    """Compile the oracle with gcc (plain C, OpenMP).  Idempotent."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _SO)
    return _SO


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build_oracle()
            lib = ctypes.CDLL(_SO)
            dp = ctypes.POINTER(ctypes.c_double)
            i64 = ctypes.c_int64
            lib.oracle_hmul.argtypes = [dp, dp, dp]
            lib.oracle_hconj.argtypes = [dp, dp]
            lib.oracle_qgemm.argtypes = [ctypes.c_char, ctypes.c_char, i64, i64, i64, dp, dp, i64,
                                         dp, i64, dp, dp, i64, ctypes.c_int]
            lib.oracle_qgemm.restype = ctypes.c_int
            lib.oracle_qgemm_entries.argtypes = [ctypes.c_char, ctypes.c_char, i64, i64, i64, dp, dp,
                                                 i64, dp, i64, dp, dp, i64, i64,
                                                 ctypes.POINTER(i64), ctypes.POINTER(i64), dp,
                                                 ctypes.c_int]
            lib.oracle_qgemm_entries.restype = ctypes.c_int
            lib.oracle_qgemv.argtypes = [ctypes.c_char, i64, i64, dp, i64, dp, dp, ctypes.c_int]
            lib.oracle_qgemv.restype = ctypes.c_int
            lib.oracle_max_threads.restype = ctypes.c_int
            _lib = lib
    return _lib


def _dptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _q(x) -> np.ndarray:
    """Scalar argument -> float64[4] quaternion (a real number r becomes (r,0,0,0))."""
    a = np.zeros(4, dtype=np.float64)
    v = np.asarray(x, dtype=np.float64).reshape(-1)
    a[: v.size] = v
    return a


def max_threads() -> int:
    return int(_load().oracle_max_threads())


def hmul(p, q) -> np.ndarray:
    """Hamilton product pq, Eq. quaternion_prod."""
    p, q = _q(p), _q(q)
    out = np.zeros(4)
    _load().oracle_hmul(_dptr(p), _dptr(q), _dptr(out))
    return out


def hconj(q) -> np.ndarray:
    """Conjugate, Eq. quaternion_conj."""
    q = _q(q)
    out = np.zeros(4)
    _load().oracle_hconj(_dptr(q), _dptr(out))
    return out


def qgemm(transA: str, transB: str, M: int, N: int, K: int, alpha, A: np.ndarray,
          B: np.ndarray, beta, C: np.ndarray, nthreads: int = 0) -> np.ndarray:
    """In place: C <- alpha op(A) op(B) + beta C (Eq. general_gemm, P:720-726;
    left scalars).  A, B, C: float64 (ncols, ld, 4)."""
    al, be = _q(alpha), _q(beta)
    lda, ldb, ldc = A.shape[1], B.shape[1], C.shape[1]
    rc = _load().oracle_qgemm(transA.encode(), transB.encode(), M, N, K, _dptr(al), _dptr(A), lda,
                              _dptr(B), ldb, _dptr(be), _dptr(C), ldc, nthreads)
    if rc != 0:
        raise ValueError(f"oracle_qgemm returned {rc}")
    return C


def qgemm_entries(transA: str, transB: str, M: int, N: int, K: int, alpha, A: np.ndarray,
                  B: np.ndarray, beta, C0: np.ndarray | None, rows, cols,
                  nthreads: int = 0) -> np.ndarray:
    """Entries (rows[s], cols[s]) of alpha op(A) op(B) + beta C0; returns (S, 4)."""
    al, be = _q(alpha), _q(beta)
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    cols = np.ascontiguousarray(cols, dtype=np.int64)
    out = np.zeros((rows.size, 4))
    if C0 is None:
        C0 = np.zeros((1, 1, 4))
    ldc = C0.shape[1]
    i64p = ctypes.POINTER(ctypes.c_int64)
    rc = _load().oracle_qgemm_entries(transA.encode(), transB.encode(), M, N, K, _dptr(al),
                                      _dptr(A), A.shape[1], _dptr(B), B.shape[1], _dptr(be),
                                      _dptr(C0), ldc, rows.size, rows.ctypes.data_as(i64p),
                                      cols.ctypes.data_as(i64p), _dptr(out), nthreads)
    if rc != 0:
        raise ValueError(f"oracle_qgemm_entries returned {rc}")
    return out


def qgemv(trans: str, rows: int, cols: int, X: np.ndarray, x: np.ndarray,
          nthreads: int = 0) -> np.ndarray:
    """y = op(X) x with x multiplied from the right; x: (cols, 4) -> y: (rows, 4)."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.zeros((rows, 4))
    rc = _load().oracle_qgemv(trans.encode(), rows, cols, _dptr(X), X.shape[1], _dptr(x),
                              _dptr(y), nthreads)
    if rc != 0:
        raise ValueError(f"oracle_qgemv returned {rc}")
    return y
