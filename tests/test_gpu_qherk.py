"""QHERK on the GPU vs the CPU oracle (-m gpu).

Reference: the oracle's full QGEMM C0' <- alpha op(A) op(A)^H + beta C0', where
C0' is C0 with the diagonal's vector part set to 0 (a Hermitian matrix has a real
diagonal; reading R18).  Checked: the `uplo` triangle within the north-star FP64
tolerance (bitwise in exact-integer mode), the diagonal's vector part exactly 0,
the other triangle and the ld padding untouched bitwise.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
import paper_1903_05575_b200 as qg
from synth import quat_matrix
from tests.gpu_helpers import path_policy
from tests.tolerance import tolerance

pytestmark = pytest.mark.gpu


def _case(N, K, uplo, trans, alpha, beta, seed, dist="uniform", pad=1, exact=False):
    rng = np.random.default_rng(seed)
    a_rows, a_cols = (N, K) if trans == "N" else (K, N)
    A = quat_matrix(rng, a_rows, a_cols, a_rows + pad, dist)
    C0 = quat_matrix(rng, N, N, N + pad, dist, pad_fill=-777.0)
    Cd = torch.from_numpy(C0).cuda()
    qg.qherk(uplo, trans, alpha, torch.from_numpy(A).cuda(), beta, Cd, N=N, K=K)
    torch.cuda.synchronize()
    got = Cd.cpu().numpy()
    ref = C0.copy()
    idx = np.arange(N)
    ref[idx, idx, 1:] = 0.0
    opA, opB = ("N", "H") if trans == "N" else ("H", "N")
    oracle.qgemm(opA, opB, N, N, K, alpha, A, A, beta, ref)
    ref[idx, idx, 1:] = 0.0
    i, j = np.meshgrid(np.arange(N), np.arange(N), indexing="ij")  # logical (row i, col j)
    tri = (i >= j) if uplo == "L" else (i <= j)
    g = got[:, :N, :].transpose(1, 0, 2)  # logical [i, j]
    r = ref[:, :N, :].transpose(1, 0, 2)
    c0 = C0[:, :N, :].transpose(1, 0, 2)
    if exact:
        np.testing.assert_array_equal(g[tri], r[tri])
    else:
        tol = tolerance("f64", K, A, a_rows, A, a_rows, (beta, 0, 0, 0), C0, N)
        assert np.abs(g[tri] - r[tri]).max() <= tol
    assert np.all(g[idx, idx, 1:] == 0.0)
    np.testing.assert_array_equal(g[~tri], c0[~tri])          # other triangle untouched
    np.testing.assert_array_equal(got[:, N:, :], C0[:, N:, :])  # padding untouched


@pytest.mark.parametrize("uplo", ["L", "U"])
@pytest.mark.parametrize("trans", ["N", "H"])
@pytest.mark.parametrize("N,K", [(1, 1), (7, 3), (64, 16), (65, 33), (130, 256), (257, 40)])
def test_qherk_ragged(uplo, trans, N, K):
    _case(N, K, uplo, trans, 0.75, -0.5, seed=N + K)


@pytest.mark.parametrize("policy", [qg.PATH_PACKED, qg.PATH_DIRECT, qg.PATH_DIRECT32],
                         ids=["packed", "direct", "direct32"])
@pytest.mark.parametrize("uplo", ["L", "U"])
@pytest.mark.parametrize("trans", ["N", "H"])
def test_qherk_exact_integer(uplo, trans, policy):
    """Bitwise in exact-integer mode on both FP64 mainloop feeds (packed chunks,
    and TMA tiles of the interleaved A with conj folded into the product signs)."""
    with path_policy(policy):
        _case(200, 70, uplo, trans, 2.0, 1.0, seed=3, dist="int8", exact=True)
        _case(130, 256, uplo, trans, 0.75, -0.5, seed=4)


@pytest.mark.parametrize("uplo", ["L", "U"])
@pytest.mark.parametrize("trans", ["N", "H"])
def test_qherk_multi_band_exact(uplo, trans):
    """N = 1297 -> 21 tile rows: two full bands of 8 tile rows of the banded
    triangle raster plus a partial band of 5, a ragged last tile row, stream-K
    over the remainder; exact-integer inputs -> bitwise."""
    _case(1297, 40, uplo, trans, 2.0, 1.0, seed=5, dist="int8", exact=True)


def test_qherk_quick_returns_and_scale():
    N, K = 40, 8
    rng = np.random.default_rng(0)
    A = torch.from_numpy(quat_matrix(rng, N, K, N)).cuda()
    C0 = quat_matrix(rng, N, N, N)
    C = torch.from_numpy(C0.copy()).cuda()
    qg.qherk("L", "N", 0.0, A, 1.0, C)          # alpha = 0, beta = 1: nothing
    assert qg.last_launch_count() == 0
    qg.qherk("U", "N", 1.0, A, 1.0, C, K=0)     # K = 0, beta = 1: nothing
    torch.cuda.synchronize()
    assert np.array_equal(C.cpu().numpy(), C0)
    qg.qherk("L", "N", 0.0, A, 0.5, C)          # C_lower <- 0.5 C_lower, diag real
    torch.cuda.synchronize()
    got = C.cpu().numpy().transpose(1, 0, 2)
    c0 = C0.transpose(1, 0, 2)
    i, j = np.meshgrid(np.arange(N), np.arange(N), indexing="ij")
    low = i > j
    np.testing.assert_array_equal(got[low], 0.5 * c0[low])
    np.testing.assert_array_equal(got[i < j], c0[i < j])
    np.testing.assert_array_equal(got[np.arange(N), np.arange(N), 0], 0.5 * c0[np.arange(N), np.arange(N), 0])
    assert np.all(got[np.arange(N), np.arange(N), 1:] == 0)


def test_qherk_c4_shape_full_size():
    """c4's shape (N = 32768, K = 256) as a Hermitian rank-K update on the lower
    triangle: sampled lower-triangle entries vs the oracle."""
    from synth.gpu_gen import counter_hermitian, counter_matrix, host_hermitian_entries
    n, K = 32768, 256
    A = counter_matrix(0, 1, n, K, "cuda")
    C = counter_hermitian(0, 3, n, "cuda")
    qg.qherk("L", "N", 1.0, A, 1.0, C)
    torch.cuda.synchronize()
    A_h = counter_matrix(0, 1, n, K, "cpu").numpy()
    rng = np.random.default_rng(9)
    r = rng.integers(0, n, 512)
    c = rng.integers(0, n, 512)
    rows, cols = np.maximum(r, c), np.minimum(r, c)          # lower triangle (row >= col)
    rows = np.concatenate([rows, np.arange(n)])
    cols = np.concatenate([cols, np.zeros(n, dtype=np.int64)])  # full first column
    t = oracle.qgemm_entries("N", "H", n, n, K, 1, A_h, A_h, 0, None, rows, cols)
    ref = t + host_hermitian_entries(0, 3, n, rows, cols)
    ref[rows == cols, 1:] = 0.0
    got = C[torch.from_numpy(cols).cuda(), torch.from_numpy(rows).cuda()].cpu().numpy()
    tol = 1e-12 * K * float(np.abs(A_h).max()) ** 2 + 8 * 2.0 ** -53 * 4
    assert np.abs(got - ref).max() <= tol
    # the strictly upper triangle still holds the input Hermitian C
    up_r, up_c = np.minimum(r, c), np.maximum(r, c)
    keep = up_r < up_c
    g_up = C[torch.from_numpy(up_c[keep]).cuda(), torch.from_numpy(up_r[keep]).cuda()].cpu().numpy()
    np.testing.assert_array_equal(g_up, host_hermitian_entries(0, 3, n, up_r[keep], up_c[keep]))
    del A, C
    torch.cuda.empty_cache()


def test_qherk_lower_and_upper_concurrently_on_one_c():
    """qherk('L') and qherk('U') into ONE C on two streams at once: each call
    touches only its own triangle (qgemm.h), so whatever the interleaving the
    strict triangles are the oracle's update -- bitwise with exact-integer inputs.
    (A diagonal tile stored whole through the TMA ring would write back the other
    triangle as it was loaded, losing the other call's update.)  The diagonal
    belongs to both calls, so it is updated once or twice depending on the race."""
    N, K = 2500, 64
    rng = np.random.default_rng(21)
    A = quat_matrix(rng, N, K, N, "int8")
    C0 = quat_matrix(rng, N, N, N, "int8")
    idx = np.arange(N)
    C0[idx, idx, 1:] = 0.0                                   # Hermitian input: real diagonal
    ref = C0.copy()
    oracle.qgemm("N", "H", N, N, K, 2.0, A, A, 1.0, ref)
    ref[idx, idx, 1:] = 0.0
    Ad = torch.from_numpy(A).cuda()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for rep in range(4):
        Cd = torch.from_numpy(C0).cuda()
        torch.cuda.synchronize()
        first, second = (("L", s1), ("U", s2)) if rep % 2 == 0 else (("U", s2), ("L", s1))
        for uplo, s in (first, second):
            with torch.cuda.stream(s):
                qg.qherk(uplo, "N", 2.0, Ad, 1.0, Cd, stream=s)
        torch.cuda.synchronize()
        got = Cd.cpu().numpy()
        off = ~np.eye(N, dtype=bool)                           # [col, row] pairs off the diagonal
        np.testing.assert_array_equal(got[off], ref[off])
        once, twice = ref[idx, idx], 2 * ref[idx, idx] - C0[idx, idx]
        d = got[idx, idx]
        assert np.all((d == once).all(axis=1) | (d == twice).all(axis=1))


def test_qherk_c4_full_triangle_every_entry_vs_oracle():
    """c4 as QHERK (N = 32768, K = 256, lower triangle) checked in full: every
    entry of the lower triangle against the oracle, column block by column block
    (rows j0.. of columns j0..j0+blk), the diagonal's vector part exactly 0 and
    the strict upper triangle bitwise equal to the input (compared on the device
    with a kept copy of C0)."""
    from synth.gpu_gen import counter_hermitian, counter_matrix
    n, K, blk = 32768, 256, 1024
    A = counter_matrix(0, 1, n, K, "cuda")
    C0 = counter_hermitian(0, 3, n, "cuda")
    C = C0.clone()
    qg.qherk("L", "N", 1.0, A, 1.0, C)
    torch.cuda.synchronize()
    A_h = counter_matrix(0, 1, n, K, "cpu").numpy()             # (K, n, 4), host generator
    tol = 1e-12 * K * float(np.abs(A_h).max()) ** 2 + 8 * 2.0 ** -53 * float(C0.abs().max()) * 4
    worst = 0.0
    rr = torch.arange(n, device="cuda").view(1, n)
    for j0 in range(0, n, blk):
        j1 = min(n, j0 + blk)
        cc = torch.arange(j0, j1, device="cuda").view(-1, 1)
        upper = rr < cc                                           # strict upper triangle of this block
        assert torch.equal(C[j0:j1][upper], C0[j0:j1][upper]), j0
        assert bool((C[j0:j1][rr == cc][:, 1:] == 0).all()), j0
        m = n - j0                                                # rows j0.. of columns j0..j1
        A_rows = np.ascontiguousarray(A_h[:, j0:, :])             # op(A) rows j0.. (stored, ld = m)
        B_blk = np.ascontiguousarray(A_h[:, j0:j1, :])            # op(B) = A^H: columns j0..j1
        ref = np.ascontiguousarray(C0[j0:j1, j0:, :].cpu().numpy())
        d = np.arange(j1 - j0)
        ref[d, d, 1:] = 0.0                                       # R18: Hermitian input, real diagonal
        oracle.qgemm("N", "H", m, j1 - j0, K, 1, A_rows, B_blk, 1, ref)
        ref[d, d, 1:] = 0.0
        got = C[j0:j1, j0:, :].cpu().numpy()
        low = np.arange(m)[None, :] >= d[:, None]                 # local row r >= local column
        worst = max(worst, float(np.abs(got[low] - ref[low]).max()))
        assert worst <= tol, (j0, worst, tol)
    del A, C0, C
    torch.cuda.empty_cache()
