"""Counter-based input generation on the device (torch int64 ops), bit-identical
to synth.inputs.counter_uniform (numpy), for the c4/c5 matrices that are too
large to draw on the host.  Holds no QGEMM arithmetic (input generation only).

Value of scalar `flat` of matrix `mid`: splitmix64(flat XOR splitmix64(key)),
key = seed * 0x100000001B3 + mid * 0x9E3779B1 (mod 2^64); top 53 bits -> u in
[0,1); value 2u - 1.  For a stored (cols, ld, 4) matrix flat = 4*(i + j*ld) + c.
"""
from __future__ import annotations

import numpy as np
import torch

from .inputs import counter_uniform  # noqa: F401  (the numpy twin; tests compare the two)

_M64 = (1 << 64) - 1


def _s64(v: int) -> int:
    v &= _M64
    return v - (1 << 64) if v >= (1 << 63) else v


def _lsr(z: torch.Tensor, s: int) -> torch.Tensor:
    return (z >> s) & ((1 << (64 - s)) - 1)


def _splitmix64_t(x: torch.Tensor) -> torch.Tensor:
    z = x + _s64(0x9E3779B97F4A7C15)
    z = (z ^ _lsr(z, 30)) * _s64(0xBF58476D1CE4E5B9)
    z = (z ^ _lsr(z, 27)) * _s64(0x94D049BB133111EB)
    return z ^ _lsr(z, 31)


def _key(seed: int, mid: int) -> int:
    k = (seed * 0x100000001B3 + mid * 0x9E3779B1) & _M64
    # splitmix64 of the key, evaluated on the host with numpy (same function)
    from .inputs import _splitmix64
    return int(_splitmix64(np.asarray(k, dtype=np.uint64)))


def counter_uniform_t(seed: int, mid: int, flat: torch.Tensor) -> torch.Tensor:
    """torch twin of counter_uniform: int64 flat indices -> float64 values."""
    hk = _s64(_key(seed, mid))
    z = _splitmix64_t(flat ^ hk)
    u = _lsr(z, 11).to(torch.float64) * (1.0 / 9007199254740992.0)
    return 2.0 * u - 1.0


def counter_normal_t(seed: int, mid: int, flat: torch.Tensor) -> torch.Tensor:
    """torch twin of synth.inputs.counter_normal (Box-Muller; device log/cos)."""
    u1 = 0.5 * (counter_uniform_t(seed, mid, 2 * flat) + 1.0)
    u2 = 0.5 * (counter_uniform_t(seed, mid, 2 * flat + 1) + 1.0)
    return torch.sqrt(-2.0 * torch.log1p(-u1)) * torch.cos((2.0 * np.pi) * u2)


def counter_block(seed: int, mid: int, ld: int, r0: int, nrows: int, c0: int, ncols: int,
                  device, dist: str = "uniform", dtype=torch.float64,
                  chunk_cols: int | None = None) -> torch.Tensor:
    """Rows [r0, r0+nrows) x columns [c0, c0+ncols) of the global stored matrix
    (leading dimension ld) whose scalar (i, j, c) is the counter draw at flat
    index 4 (i + j ld) + c, generated on `device` as a compact (ncols, nrows, 4)
    tensor: a rank's row block of a sharded matrix, or a column panel, without
    materialising the rest (synth.inputs.counter_block_host is the numpy twin)."""
    out = torch.empty((ncols, nrows, 4), dtype=dtype, device=device)
    if ncols == 0 or nrows == 0:
        return out
    gen = counter_uniform_t if dist == "uniform" else counter_normal_t
    step = chunk_cols or max(1, (1 << 25) // max(1, 4 * nrows))
    i = torch.arange(r0, r0 + nrows, dtype=torch.int64, device=device).view(1, -1, 1)
    c = torch.arange(4, dtype=torch.int64, device=device).view(1, 1, 4)
    for j0 in range(0, ncols, step):
        j1 = min(ncols, j0 + step)
        j = torch.arange(c0 + j0, c0 + j1, dtype=torch.int64, device=device).view(-1, 1, 1)
        out[j0:j1] = gen(seed, mid, 4 * (i + j * ld) + c).to(dtype)
    return out


def counter_matrix(seed: int, mid: int, rows: int, cols: int, device, dtype=torch.float64,
                   chunk: int = 1 << 26) -> torch.Tensor:
    """Stored rows x cols matrix (cols, rows, 4) (ld = rows) from the counter generator."""
    out = torch.empty((cols, rows, 4), dtype=dtype, device=device)
    flat_out = out.view(-1)
    n = flat_out.numel()
    for s in range(0, n, chunk):
        e = min(n, s + chunk)
        idx = torch.arange(s, e, dtype=torch.int64, device=device)
        flat_out[s:e] = counter_uniform_t(seed, mid, idx).to(dtype)
    return out


def counter_hermitian(seed: int, mid: int, n: int, device, chunk_cols: int = 512, r0: int = 0,
                      nrows: int | None = None) -> torch.Tensor:
    """C = (X + X^H)/2 with X the counter matrix (seed, mid), n x n, ld = n
    (reading R14).  Entry (i, j): (X_ij + conj(X_ji)) / 2, computed from the
    counter directly (no X materialised).  Rows [r0, r0 + nrows) only (default:
    all), as a compact (n, nrows, 4) tensor: a rank's row block."""
    nrows = n - r0 if nrows is None else nrows
    out = torch.empty((n, nrows, 4), dtype=torch.float64, device=device)
    i = torch.arange(r0, r0 + nrows, dtype=torch.int64, device=device).view(1, nrows, 1)
    c = torch.arange(4, dtype=torch.int64, device=device).view(1, 1, 4)
    sign = torch.tensor([1.0, -1.0, -1.0, -1.0], dtype=torch.float64, device=device)
    for j0 in range(0, n, chunk_cols):
        j1 = min(n, j0 + chunk_cols)
        j = torch.arange(j0, j1, dtype=torch.int64, device=device).view(-1, 1, 1)
        x_ij = counter_uniform_t(seed, mid, 4 * (i + j * n) + c)
        x_ji = counter_uniform_t(seed, mid, 4 * (j + i * n) + c)
        out[j0:j1] = 0.5 * (x_ij + sign * x_ji)
    return out


# ---------------------------------------------------------------- host samplers (numpy)
def host_rows_N(seed: int, mid: int, ld: int, rows: np.ndarray, ncols: int) -> np.ndarray:
    """Rows `rows` of a stored column-major matrix, as a stored (ncols, len(rows), 4) array."""
    r = np.asarray(rows, dtype=np.int64).reshape(1, -1, 1)
    j = np.arange(ncols, dtype=np.int64).reshape(-1, 1, 1)
    c = np.arange(4, dtype=np.int64).reshape(1, 1, 4)
    return counter_uniform(seed, mid, 4 * (r + j * ld) + c)


def host_cols(seed: int, mid: int, ld: int, cols: np.ndarray, nrows: int) -> np.ndarray:
    """Columns `cols` (first nrows rows) of a stored matrix: (len(cols), nrows, 4)."""
    j = np.asarray(cols, dtype=np.int64).reshape(-1, 1, 1)
    r = np.arange(nrows, dtype=np.int64).reshape(1, -1, 1)
    c = np.arange(4, dtype=np.int64).reshape(1, 1, 4)
    return counter_uniform(seed, mid, 4 * (r + j * ld) + c)


def host_hermitian_entries(seed: int, mid: int, n: int, rows, cols) -> np.ndarray:
    """(X_ij + conj(X_ji))/2 at the given (i, j) pairs: (S, 4)."""
    i = np.asarray(rows, dtype=np.int64).reshape(-1, 1)
    j = np.asarray(cols, dtype=np.int64).reshape(-1, 1)
    c = np.arange(4, dtype=np.int64).reshape(1, 4)
    x_ij = counter_uniform(seed, mid, 4 * (i + j * n) + c)
    x_ji = counter_uniform(seed, mid, 4 * (j + i * n) + c)
    return 0.5 * (x_ij + np.array([1.0, -1.0, -1.0, -1.0]) * x_ji)
