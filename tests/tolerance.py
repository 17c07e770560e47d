"""Parity tolerances (BASELINE.json north_star), with DESIGN.md reading R8.

FP64: max|C - C_ref| <= 1e-12 * K * max|A| * max|B|
FP32: max|C - C_ref| <= 1e-4 * sqrt(K) * max|A| * max|B|
max|A|, max|B| = max absolute REAL COMPONENT over the logical operand (padding
excluded).  Reading R8 adds 8 u |beta| max|C0| (u = unit roundoff) so that the
beta*C0 term, evaluated with different FMA contraction on CPU and GPU, is
covered when the main term vanishes (alpha = 0, K = 0).
"""
from __future__ import annotations

import math

import numpy as np


def _maxabs_stored(X: np.ndarray, rows: int) -> float:
    if X is None or X.size == 0 or rows == 0:
        return 0.0
    v = X[:, :rows, :]
    return float(np.max(np.abs(v))) if v.size else 0.0


def tolerance(precision: str, K: int, A, a_rows: int, B, b_rows: int, beta=None, C0=None,
              c_rows: int = 0) -> float:
    ma = _maxabs_stored(A, a_rows)
    mb = _maxabs_stored(B, b_rows)
    if precision == "f64":
        t = 1e-12 * K * ma * mb
        u = 2.0 ** -53
    elif precision == "f32":
        t = 1e-4 * math.sqrt(K) * ma * mb
        u = 2.0 ** -24
    else:
        raise ValueError(precision)
    if beta is not None and C0 is not None:
        nb = float(np.linalg.norm(np.asarray(beta, dtype=np.float64)))
        if nb != 0.0:
            t += 8 * u * nb * _maxabs_stored(C0, c_rows) * 4
    return t
