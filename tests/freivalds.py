"""Block Freivalds check of a full-size QGEMM result (tests only).

Over the quaternions matrix multiplication is associative, so for any
right operand X

    C X  ==  alpha op(A) (op(B) X) + beta C0 X          (exactly, in real arithmetic)

and a residual R = C X - (alpha op(A) (op(B) X) + beta C0 X) far above rounding
level flags a wrong C.  X here is block-diagonal: vector v is supported on the
column block J_v = [v bs, (v+1) bs) of C with quaternion entries x_j of norm in
[1, 2] (random direction), so

    R[i, v] = sum_{j in J_v} (C_ij - C*_ij) x_j   (+ rounding of the check itself),

and a single wrong entry C_ij = C*_ij + d moves R[i, v(j)] by d x_j, of norm
|d| |x_j| >= |d| (norm multiplicativity).  Short blocks keep the
rounding noise of the other bs - 1 terms small (it grows like sqrt(bs)).

Every product is an oracle call (oracle.qgemv / oracle.qgemm); no CUDA-path value
enters the right-hand side.  The pass bound is CALIBRATED on rows whose exact
result is known from the oracle (the sampled full rows): the residual of the
oracle's own C on those rows, and of the GPU's C on those rows (verified entry by
entry against the per-entry tolerance), give the noise level; the bound is
CAL_FACTOR times that (<= 1e3 times the correct-C residual).
"""
from __future__ import annotations

from typing import Callable

import numpy as np

import oracle

CAL_FACTOR = 20.0


def qnorm(r: np.ndarray) -> np.ndarray:
    """Quaternion norms of (..., 4) arrays."""
    return np.sqrt((r * r).sum(axis=-1))


def draw_x(n: int, seed: int) -> np.ndarray:
    """n quaternions of norm in [1, 2] with uniformly random direction: (n, 4)."""
    rng = np.random.default_rng(seed)
    d = rng.standard_normal((n, 4))
    d /= qnorm(d)[:, None]
    return d * rng.uniform(1.0, 2.0, size=(n, 1))


def blocks(n: int, bs: int):
    return [(j0, min(n, j0 + bs)) for j0 in range(0, n, bs)]


def times_x(get_block: Callable[[int, int], tuple[np.ndarray, str]], rows: int, n: int,
            x: np.ndarray, bs: int) -> np.ndarray:
    """Y[:, v] = sum_{j in J_v} op(X)[:, j] x_j for an operand whose columns j0..j1
    get_block returns as (stored array, op) with op(stored) = rows x (j1 - j0);
    result stored (nb, rows, 4)."""
    bl = blocks(n, bs)
    out = np.zeros((len(bl), rows, 4))
    for v, (j0, j1) in enumerate(bl):
        X, op = get_block(j0, j1)
        out[v] = oracle.qgemv(op, rows, j1 - j0, np.ascontiguousarray(X), x[j0:j1])
    return out


def columns_of(X: np.ndarray):
    """get_block for a stored matrix used as is (op N): columns j0..j1."""
    return lambda j0, j1: (X[j0:j1], "N")


class Check:
    """R = C X - alpha op(A) (op(B) X) - beta C0 X, with the noise calibration.

    rhs: the oracle's alpha op(A) (op(B) X) + beta C0 X, (nb, M, 4).
    """

    def __init__(self, M: int, n: int, bs: int, x: np.ndarray, rhs: np.ndarray):
        self.M, self.n, self.bs, self.x, self.rhs = M, n, bs, x, rhs

    def residual(self, get_c_block) -> np.ndarray:
        return times_x(get_c_block, self.M, self.n, self.x, self.bs) - self.rhs

    def residual_rows(self, C_rows_st: np.ndarray, rows: np.ndarray) -> np.ndarray:
        """Residual on selected rows whose full C row is given stored as
        (N, len(rows), 4) (columns of the row sample)."""
        cx = times_x(columns_of(C_rows_st), len(rows), self.n, self.x, self.bs)
        return cx - self.rhs[:, rows, :]

    def bound(self, ref_rows_st: np.ndarray, got_rows_st: np.ndarray, rows: np.ndarray,
              factor: float = CAL_FACTOR) -> float:
        """`factor` x the largest residual norm on the sampled rows, of the
        oracle's C (the correct-C residual) and of the GPU's verified rows."""
        noise = max(float(qnorm(self.residual_rows(ref_rows_st, rows)).max()),
                    float(qnorm(self.residual_rows(got_rows_st, rows)).max()))
        return factor * noise


def detects(bound: float, tol: float, factor: float) -> bool:
    """Power of the check: an entry off by 10 tol moves its residual by >= 10 tol
    (|x_j| >= 1); the other bs - 1 terms of that residual add at most the noise
    level ~ bound / factor, so the entry is caught if 10 tol - bound/factor > bound."""
    return bound * (1.0 + 1.0 / factor) < 10.0 * tol
