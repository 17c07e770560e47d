"""Complex-block (SU(2)) embedding chi of quaternion matrices, numpy only.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

chi(Q) = Q^0 (x) sigma_0 + Q^1 (x) i sigma_3 + Q^2 (x) i sigma_2 + Q^3 (x) i sigma_1
       = [[ U0,        U1       ],
          [ -conj(U1), conj(U0) ]],   U0 = Q^0 + i Q^1,  U1 = Q^2 + i Q^3
(Eq. qmat_complex; scalar form Eq. h_matrep), laid out
blockwise as displayed.  chi is an algebra homomorphism,
PQ <-> chi(P) chi(Q) (Eq. hc_mat_mult), so a *library* complex GEMM
(numpy matmul -> host ZGEMM) on the 2M x 2N embedding gives an independent
check of every sign of the quaternion product.

Logical matrices here are numpy arrays of shape (rows, cols, 4): entry
[i, j, c] is component c of X_{ij}.  ``storage_to_logical`` converts from the
(ncols, ld, 4) column-major storage layout.
"""
from __future__ import annotations

import numpy as np


def storage_to_logical(X: np.ndarray, rows: int) -> np.ndarray:
    """(ncols, ld, 4) column-major storage -> (rows, ncols, 4) logical view copy."""
    return np.ascontiguousarray(X[:, :rows, :].transpose(1, 0, 2))


def logical_to_storage(L: np.ndarray, ld: int | None = None, fill=np.nan) -> np.ndarray:
    rows, cols = L.shape[:2]
    ld = rows if ld is None else ld
    X = np.full((cols, ld, 4), fill, dtype=L.dtype)
    X[:, :rows, :] = L.transpose(1, 0, 2)
    return X


def op_materialise(op: str, L: np.ndarray) -> np.ndarray:
    """op(X) of a logical matrix: 'N' -> X, 'T' -> X^T, 'H'/'C' -> X^H."""
    op = op.upper()
    if op == "N":
        return L.copy()
    T = np.ascontiguousarray(L.transpose(1, 0, 2))
    if op == "T":
        return T
    if op in ("H", "C"):
        T[..., 1:] *= -1.0  # conj of each entry, Eq. quaternion_conj
        return T
    raise ValueError(op)


def chi(L: np.ndarray) -> np.ndarray:
    """Quaternion logical matrix (m, n, 4) -> complex128 (2m, 2n), Eq. qmat_complex."""
    U0 = L[..., 0] + 1j * L[..., 1]
    U1 = L[..., 2] + 1j * L[..., 3]
    return np.block([[U0, U1], [-np.conj(U1), np.conj(U0)]])


def unchi(Z: np.ndarray) -> np.ndarray:
    """Inverse of chi on its image: read Q back from the top block row."""
    m2, n2 = Z.shape
    m, n = m2 // 2, n2 // 2
    U0, U1 = Z[:m, :n], Z[:m, n:]
    out = np.empty((m, n, 4))
    out[..., 0], out[..., 1] = U0.real, U0.imag
    out[..., 2], out[..., 3] = U1.real, U1.imag
    return out


def chi_scalar(q) -> np.ndarray:
    """2x2 complex representation of a quaternion scalar, Eq. h_matrep."""
    return chi(np.asarray(q, dtype=np.float64).reshape(1, 1, 4))


def _q4(x) -> np.ndarray:
    a = np.zeros(4)
    v = np.asarray(x, dtype=np.float64).reshape(-1)
    a[: v.size] = v
    return a


def reference_gemm_via_chi(opA: str, opB: str, alpha, LA: np.ndarray, LB: np.ndarray, beta,
                           LC: np.ndarray | None) -> np.ndarray:
    """alpha op(A) op(B) + beta C evaluated entirely in the complex embedding with
    numpy matmul (library ZGEMM).  Left scalars become left products with the
    embedded diagonal matrices diag(alpha).  Independent of the C
    oracle: shares no arithmetic with it."""
    PA, PB = op_materialise(opA, LA), op_materialise(opB, LB)
    m, n = PA.shape[0], PB.shape[1]
    T = chi(PA) @ chi(PB)
    Da = chi(_q4(alpha)[None, None, :] * np.eye(m)[..., None])
    out = Da @ T
    b = _q4(beta)
    if LC is not None and np.any(b != 0):
        Db = chi(b[None, None, :] * np.eye(m)[..., None])
        out = out + Db @ chi(LC)
    assert out.shape == (2 * m, 2 * n)
    return unchi(out)
