"""Seeded synthetic QGEMM problems (recipes in DESIGN.md §"Input recipe").

Storage layout: a numpy array of shape (ncols, ld, 4), C-contiguous, is the
column-major interleaved layout of include/qgemm.h (element (i, j) component c
at flat index 4*(i + j*ld) + c).

Readings: seed 0 for reported runs, {0,1,2} in tests; draw order
A, B, C; uniform[-1,1] is 2u-1 with u = Generator.random() in [0,1) (R13);
"Hermitian-quaternion initialised" C is (X + X^H)/2 with X uniform (R14).
The paper's own workload is square random matrices of unstated distribution
(P:1616-1618); BASELINE.json's five configs stand in for it.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

# BASELINE.json "configs", restated as parameters.
CONFIGS = {
    "c1": dict(M=64, N=64, K=64, ops=[("N", "N")], alpha=(1, 0, 0, 0), beta=(0, 0, 0, 0),
               dist="uniform", ld_pad=0, dtype="f64"),
    "c2": dict(M=1024, N=1024, K=1024,
               ops=[(a, b) for a in "NTH" for b in "NTH"],
               alpha=(0.75, 0, 0, 0), beta=(-0.5, 0, 0, 0), dist="uniform", ld=1040,
               dtype="f64"),
    "c3": dict(M=8192, N=8192, K=8192, ops=[("N", "H")], alpha=(1, 0, 0, 0),
               beta=(1, 0, 0, 0), dist="normal", ld_pad=0, dtype="f64+f32"),
    "c4": dict(M=32768, N=32768, K=256, ops=[("N", "H")], alpha=(1, 0, 0, 0),
               beta=(1, 0, 0, 0), dist="uniform", c_init="hermitian", b_is_a=True,
               ld_pad=0, dtype="f64"),
    "c5": dict(M=32768, N=32768, K=32768, ops=[("N", "N")], alpha=(1, 0, 0, 0),
               beta=(0, 0, 0, 0), dist="uniform", c_init="nan", ld_pad=0, dtype="f64"),
}


def stored_shape(op: str, rows: int, cols: int) -> tuple[int, int]:
    """Stored (nrows, ncols) of X such that op(X) is rows x cols."""
    return (rows, cols) if op.upper() == "N" else (cols, rows)


def _draw(rng: np.random.Generator, n: int, dist: str) -> np.ndarray:
    if dist == "uniform":
        return 2.0 * rng.random(n) - 1.0
    if dist == "normal":
        return rng.standard_normal(n)
    if dist == "int8":  # exact-integer mode: components in [-8, 8]
        return rng.integers(-8, 9, size=n).astype(np.float64)
    if dist == "int2":
        return rng.integers(-2, 3, size=n).astype(np.float64)
    raise ValueError(dist)


def quat_matrix(rng: np.random.Generator, rows: int, cols: int, ld: int | None = None,
                dist: str = "uniform", pad_fill: float = np.nan,
                dtype=np.float64) -> np.ndarray:
    """Stored rows x cols quaternion matrix, (cols, ld, 4); ld padding = pad_fill."""
    ld = max(1, rows) if ld is None else ld
    assert ld >= max(1, rows)
    X = np.full((max(cols, 0), ld, 4), pad_fill, dtype=np.float64)
    if rows > 0 and cols > 0:
        X[:, :rows, :] = _draw(rng, rows * cols * 4, dist).reshape(cols, rows, 4)
    return X.astype(dtype, copy=False)


def hermitian_matrix(rng: np.random.Generator, n: int, ld: int | None = None,
                     dist: str = "uniform", pad_fill: float = np.nan) -> np.ndarray:
    """(X + X^H)/2 stored as (n, ld, 4): real diagonal, C_ji = conj(C_ij) (reading R14)."""
    X = quat_matrix(rng, n, n, n, dist)
    L = X.transpose(1, 0, 2)  # logical [i, j, c]
    LH = L.transpose(1, 0, 2).copy()
    LH[..., 1:] *= -1.0
    H = 0.5 * (L + LH)
    ld = n if ld is None else ld
    out = np.full((n, ld, 4), pad_fill)
    out[:, :n, :] = H.transpose(1, 0, 2)
    return out


# ----------------------------------------------------------------------------
# Counter-based generator for inputs too large to draw on the host
# (SURVEY §8(d)): u(seed, matrix_id, flat index) via splitmix64 -> 53 bits.
# ----------------------------------------------------------------------------
_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def counter_uniform(seed: int, matrix_id: int, flat_index: np.ndarray) -> np.ndarray:
    """uniform[-1,1) value of scalar `flat_index` of matrix `matrix_id`."""
    idx = np.asarray(flat_index, dtype=np.uint64)
    with np.errstate(over="ignore"):
        key = np.uint64((seed * 0x100000001B3 + matrix_id * 0x9E3779B1) & 0xFFFFFFFFFFFFFFFF)
        z = _splitmix64(idx ^ _splitmix64(np.asarray(key, dtype=np.uint64)))
    u = (z >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    return 2.0 * u - 1.0


def counter_normal(seed: int, matrix_id: int, flat_index: np.ndarray) -> np.ndarray:
    """Standard normal value of scalar `flat_index` of matrix `matrix_id`:
    Box-Muller on two counter draws (u1, u2) at counters 2f and 2f+1,
    z = sqrt(-2 ln(1 - u1)) cos(2 pi u2)  (1 - u1 in (0, 1], so the log is finite).
    Its torch twin (synth.gpu_gen.counter_normal_t) uses the device's log/cos:
    equal to a few ulp, not bitwise."""
    f = np.asarray(flat_index, dtype=np.uint64)
    with np.errstate(over="ignore"):
        u1 = 0.5 * (counter_uniform(seed, matrix_id, f * np.uint64(2)) + 1.0)
        u2 = 0.5 * (counter_uniform(seed, matrix_id, f * np.uint64(2) + np.uint64(1)) + 1.0)
    return np.sqrt(-2.0 * np.log1p(-u1)) * np.cos(2.0 * np.pi * u2)


def counter_gather_host(seed: int, matrix_id: int, ld: int, rows, cols,
                        dist: str = "uniform") -> np.ndarray:
    """Entries (rows x cols) of the stored matrix whose scalar (i, j, c) is the
    counter draw at flat index 4 (i + j ld) + c, as a compact (len(cols),
    len(rows), 4) array: the sampled rows / columns a parity check needs."""
    i = np.asarray(rows, dtype=np.int64).reshape(1, -1, 1)
    j = np.asarray(cols, dtype=np.int64).reshape(-1, 1, 1)
    c = np.arange(4, dtype=np.int64).reshape(1, 1, 4)
    flat = 4 * (i + j * ld) + c
    return (counter_uniform if dist == "uniform" else counter_normal)(seed, matrix_id, flat)


def counter_block_host(seed: int, matrix_id: int, ld: int, r0: int, nrows: int, c0: int,
                       ncols: int, dist: str = "uniform") -> np.ndarray:
    """Rows [r0, r0+nrows) x columns [c0, c0+ncols) (counter_gather_host)."""
    return counter_gather_host(seed, matrix_id, ld, np.arange(r0, r0 + nrows),
                               np.arange(c0, c0 + ncols), dist)


@dataclass
class Problem:
    """One QGEMM call: C <- alpha op(A) op(B) + beta C (stored numpy arrays)."""
    transA: str
    transB: str
    M: int
    N: int
    K: int
    alpha: np.ndarray
    beta: np.ndarray
    A: np.ndarray
    B: np.ndarray
    C: np.ndarray
    meta: dict = field(default_factory=dict)

    @property
    def flops(self) -> float:
        return 32.0 * self.M * self.N * self.K  # 16 real FMAs per quaternion MAC (Table 1)


def make_problem(M: int, N: int, K: int, transA: str = "N", transB: str = "N",
                 alpha=(1, 0, 0, 0), beta=(0, 0, 0, 0), seed: int = 0, dist: str = "uniform",
                 lda: int | None = None, ldb: int | None = None, ldc: int | None = None,
                 c_init: str = "random", b_is_a: bool = False,
                 pad_fill: float = np.nan, c_pad_fill: float = -7777.0) -> Problem:
    """Draw A, B, C (in that order) from default_rng(seed)."""
    rng = np.random.default_rng(seed)
    ar, ac = stored_shape(transA, M, K)
    br, bc = stored_shape(transB, K, N)
    A = quat_matrix(rng, ar, ac, lda if lda is not None else max(1, ar), dist, pad_fill)
    if b_is_a:
        B = A
    else:
        B = quat_matrix(rng, br, bc, ldb if ldb is not None else max(1, br), dist, pad_fill)
    ldc_ = ldc if ldc is not None else max(1, M)
    if c_init == "random":
        C = quat_matrix(rng, M, N, ldc_, dist, c_pad_fill)
    elif c_init == "hermitian":
        assert M == N
        C = hermitian_matrix(rng, M, ldc_, dist, c_pad_fill)
    elif c_init == "nan":
        C = np.full((N, ldc_, 4), np.nan)
        C[:, M:, :] = c_pad_fill
    elif c_init == "zero":
        C = np.zeros((N, ldc_, 4))
        C[:, M:, :] = c_pad_fill
    else:
        raise ValueError(c_init)
    al = np.zeros(4); al[: len(np.atleast_1d(alpha))] = np.atleast_1d(alpha)
    be = np.zeros(4); be[: len(np.atleast_1d(beta))] = np.atleast_1d(beta)
    return Problem(transA, transB, M, N, K, al, be, A, B, C,
                   dict(seed=seed, dist=dist, c_init=c_init))
