"""Pins of the CPU oracle against what the paper and mathematics fix (-m "not gpu").

Each test names the PAPER.md passage ("P:n") it pins.  None of them re-types
the oracle's formula: the expected values come from hand-evaluated golden
files, the paper's Pauli map, library routines (numpy complex / real matmul
on the chi-embedding), algebraic identities, or exact integer arithmetic.
"""
from __future__ import annotations

import os

import numpy as np
import pytest

import oracle
from oracle.embedding import (chi, chi_scalar, logical_to_storage, op_materialise,
                              reference_gemm_via_chi, storage_to_logical, unchi)
from synth import make_problem, quat_matrix

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
OPS = [(a, b) for a in "NTH" for b in "NTH"]


def _read_table(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            rows.append([part.split() for part in line.split("|")])
    return rows


# ---------------------------------------------------------------- scalar pins
def test_basis_table_exact():
    """P1: all 16 e_p e_s from Eq. quaternion_alg, exact."""
    rows = _read_table("basis_table.txt")
    assert len(rows) == 16
    for (ps, r) in rows:
        p, s = int(ps[0]), int(ps[1])
        ep = np.eye(4)[p]
        es = np.eye(4)[s]
        np.testing.assert_array_equal(oracle.hmul(ep, es), np.array(r, dtype=float))


def test_e1e2e3_is_minus_e0():
    """e1 e2 e3 = -e0, and e_i e_j = -e_j e_i."""
    e = np.eye(4)
    np.testing.assert_array_equal(oracle.hmul(oracle.hmul(e[1], e[2]), e[3]), -e[0])
    np.testing.assert_array_equal(oracle.hmul(e[1], oracle.hmul(e[2], e[3])), -e[0])
    for i in (1, 2, 3):
        for j in (1, 2, 3):
            if i != j:
                np.testing.assert_array_equal(oracle.hmul(e[i], e[j]), -oracle.hmul(e[j], e[i]))


def test_worked_products_exact():
    """P2: hand-evaluated products (golden/worked_products.txt), exact."""
    for label, p, q, r in _read_table("worked_products.txt"):
        np.testing.assert_array_equal(oracle.hmul(np.array(p, float), np.array(q, float)),
                                      np.array(r, float), err_msg=label[0])


def test_conjugate():
    """Eq. quaternion_conj and the golden conj products."""
    np.testing.assert_array_equal(oracle.hconj([1, 2, 3, 4]), [1, -2, -3, -4])
    np.testing.assert_array_equal(oracle.hconj(oracle.hconj([1.5, -2, 3, 4])), [1.5, -2, 3, 4])


def test_norm_multiplicative():
    """P3: normed division algebra: |pq| = |p||q|, relative 1e-14."""
    rng = np.random.default_rng(1)
    for _ in range(200):
        p = rng.standard_normal(4) * 10.0 ** rng.uniform(-3, 3)
        q = rng.standard_normal(4) * 10.0 ** rng.uniform(-3, 3)
        lhs = np.linalg.norm(oracle.hmul(p, q))
        rhs = np.linalg.norm(p) * np.linalg.norm(q)
        assert abs(lhs - rhs) <= 1e-14 * rhs


def test_conj_antihomomorphism():
    """conj(pq) = conj(q) conj(p)."""
    rng = np.random.default_rng(2)
    for _ in range(100):
        p, q = rng.standard_normal(4), rng.standard_normal(4)
        lhs = oracle.hconj(oracle.hmul(p, q))
        rhs = oracle.hmul(oracle.hconj(q), oracle.hconj(p))
        np.testing.assert_allclose(lhs, rhs, rtol=0, atol=4e-15 * np.abs(p).sum() * np.abs(q).sum())


def test_pauli_map():
    """chi on the basis equals the paper's Pauli map e0->s0, e1->i s3, e2->i s2, e3->i s1
    (P:393-403), pinning the embedding itself."""
    s0 = np.eye(2)
    s1 = np.array([[0, 1], [1, 0]])
    s2 = np.array([[0, -1j], [1j, 0]])
    s3 = np.array([[1, 0], [0, -1]])
    e = np.eye(4)
    np.testing.assert_array_equal(chi_scalar(e[0]), s0)
    np.testing.assert_array_equal(chi_scalar(e[1]), 1j * s3)
    np.testing.assert_array_equal(chi_scalar(e[2]), 1j * s2)
    np.testing.assert_array_equal(chi_scalar(e[3]), 1j * s1)


def test_hmul_vs_complex_2x2():
    """P6 (scalar): pq <-> chi(p) chi(q), Eq. hc_mult, library 2x2 matmul."""
    rng = np.random.default_rng(3)
    for _ in range(200):
        p, q = rng.standard_normal(4), rng.standard_normal(4)
        got = chi_scalar(oracle.hmul(p, q))
        ref = chi_scalar(p) @ chi_scalar(q)
        np.testing.assert_allclose(got, ref, rtol=0, atol=1e-14 * (1 + np.abs(ref).max()))


# ---------------------------------------------------------------- matrix pins
@pytest.mark.parametrize("opA,opB", OPS)
def test_qgemm_vs_complex_embedding(opA, opB):
    """P6: oracle QGEMM vs numpy complex GEMM on the 2M x 2N chi-embedding
    (Eq. qmat_complex, Eq. hc_mat_mult) for all 9 op pairs,
    with quaternion alpha/beta from the left and NaN ld padding."""
    M, N, K = 7, 5, 6
    alpha = np.array([0.3, -1.2, 0.7, 0.25])
    beta = np.array([-0.5, 0.1, -0.9, 0.4])
    pr = make_problem(M, N, K, opA, opB, alpha, beta, seed=11,
                      lda=(M if opA == "N" else K) + 3, ldb=(K if opB == "N" else N) + 2,
                      ldc=M + 4)
    C0 = pr.C.copy()
    oracle.qgemm(opA, opB, M, N, K, alpha, pr.A, pr.B, beta, pr.C)
    LA = storage_to_logical(pr.A, M if opA == "N" else K)
    LB = storage_to_logical(pr.B, K if opB == "N" else N)
    LC0 = storage_to_logical(C0, M)
    ref = reference_gemm_via_chi(opA, opB, alpha, LA, LB, beta, LC0)
    got = storage_to_logical(pr.C, M)
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-13)
    # padding of C untouched
    np.testing.assert_array_equal(pr.C[:, M:, :], C0[:, M:, :])


@pytest.mark.parametrize("opA,opB", OPS)
def test_exact_integer_mode_bitwise(opA, opB):
    """P8: integer components in [-8, 8]: every partial sum is an exact integer,
    so the oracle must equal the complex-embedding GEMM BITWISE."""
    M, N, K = 9, 6, 17
    pr = make_problem(M, N, K, opA, opB, (2, -1, 0, 3), (1, 0, -2, 1), seed=5, dist="int8")
    C0 = pr.C.copy()
    oracle.qgemm(opA, opB, M, N, K, pr.alpha, pr.A, pr.B, pr.beta, pr.C)
    ref = reference_gemm_via_chi(opA, opB, pr.alpha,
                                 storage_to_logical(pr.A, M if opA == "N" else K),
                                 storage_to_logical(pr.B, K if opB == "N" else N),
                                 pr.beta, storage_to_logical(C0, M))
    np.testing.assert_array_equal(storage_to_logical(pr.C, M), ref)


def test_associativity():
    """P4: (AB)C = A(BC) (P:318-320 associativity of H carried to matrices)."""
    rng = np.random.default_rng(4)
    A = quat_matrix(rng, 3, 5)
    B = quat_matrix(rng, 5, 2)
    Cm = quat_matrix(rng, 2, 4)
    AB = np.zeros((2, 3, 4))
    oracle.qgemm("N", "N", 3, 2, 5, 1, A, B, 0, AB)
    L = np.zeros((4, 3, 4))
    oracle.qgemm("N", "N", 3, 4, 2, 1, AB, Cm, 0, L)
    BC = np.zeros((4, 5, 4))
    oracle.qgemm("N", "N", 5, 4, 2, 1, B, Cm, 0, BC)
    R = np.zeros((4, 3, 4))
    oracle.qgemm("N", "N", 3, 4, 5, 1, A, BC, 0, R)
    np.testing.assert_allclose(L, R, rtol=0, atol=1e-13 * np.abs(R).max())


def test_conjugate_transpose_of_product():
    """P5: (AB)^H = B^H A^H, using op='H' on both."""
    rng = np.random.default_rng(6)
    M, N, K = 6, 4, 5
    A = quat_matrix(rng, M, K)
    B = quat_matrix(rng, K, N)
    AB = np.zeros((N, M, 4))
    oracle.qgemm("N", "N", M, N, K, 1, A, B, 0, AB)
    BhAh = np.zeros((M, N, 4))   # N x M result, stored (M cols, ld N)
    oracle.qgemm("H", "H", N, M, K, 1, B, A, 0, BhAh)
    lhs = op_materialise("H", storage_to_logical(AB, M))
    np.testing.assert_allclose(storage_to_logical(BhAh, N), lhs, rtol=0, atol=1e-14)


def test_transpose_is_not_antihomomorphic():
    """A5: (AB)^T != B^T A^T over H (non-commutativity): the op='T'
    path must not be implemented as a transpose swap."""
    rng = np.random.default_rng(7)
    A = quat_matrix(rng, 3, 5)
    B = quat_matrix(rng, 5, 2)
    AB = np.zeros((2, 3, 4))
    oracle.qgemm("N", "N", 3, 2, 5, 1, A, B, 0, AB)
    BtAt = np.zeros((3, 2, 4))
    oracle.qgemm("T", "T", 2, 3, 5, 1, B, A, 0, BtAt)
    lhs = op_materialise("T", storage_to_logical(AB, 3))
    assert np.abs(storage_to_logical(BtAt, 2) - lhs).max() > 0.1


def test_complex_subalgebra_matches_complex_gemm():
    """P7: Q^2 = Q^3 = 0 (Eq. complex_subalg_mat): QGEMM == ZGEMM of
    Q^0 + i Q^1 (Eq. h_c_mat_iso), components 2,3 exactly zero."""
    rng = np.random.default_rng(8)
    M, N, K = 8, 7, 9
    A = quat_matrix(rng, M, K); A[..., 2:] = 0
    B = quat_matrix(rng, K, N); B[..., 2:] = 0
    C = np.zeros((N, M, 4))
    oracle.qgemm("N", "N", M, N, K, 1, A, B, 0, C)
    ZA = storage_to_logical(A, M)[..., 0] + 1j * storage_to_logical(A, M)[..., 1]
    ZB = storage_to_logical(B, K)[..., 0] + 1j * storage_to_logical(B, K)[..., 1]
    Z = ZA @ ZB
    L = storage_to_logical(C, M)
    np.testing.assert_allclose(L[..., 0] + 1j * L[..., 1], Z, rtol=0, atol=1e-14 * K)
    assert np.all(L[..., 2:] == 0)


def test_real_subalgebra_matches_real_gemm():
    """P7: Q^1 = Q^2 = Q^3 = 0: QGEMM == DGEMM on Q^0."""
    rng = np.random.default_rng(9)
    M, N, K = 6, 9, 4
    A = quat_matrix(rng, M, K); A[..., 1:] = 0
    B = quat_matrix(rng, K, N); B[..., 1:] = 0
    C = np.zeros((N, M, 4))
    oracle.qgemm("N", "N", M, N, K, 1, A, B, 0, C)
    ref = storage_to_logical(A, M)[..., 0] @ storage_to_logical(B, K)[..., 0]
    L = storage_to_logical(C, M)
    np.testing.assert_allclose(L[..., 0], ref, rtol=0, atol=1e-14 * K)
    assert np.all(L[..., 1:] == 0)


# ---------------------------------------------------------------- closed forms
def _golden_products():
    return {r[0][0]: (np.array(r[1], float), np.array(r[2], float), np.array(r[3], float))
            for r in _read_table("worked_products.txt")}


@pytest.mark.parametrize("opA,opB,label", [("N", "N", "pq"), ("N", "H", "p_conjq"),
                                           ("H", "N", "conjp_q"), ("T", "T", "pq")])
def test_constant_matrices_closed_form(opA, opB, label):
    """P9: A == p, B == q (constant) => C_ij = K (op p)(op q) exactly, with the
    hand-evaluated products of golden/worked_products.txt."""
    g = _golden_products()
    p = np.array([1.0, 2, 3, 4]); q = np.array([5.0, 6, 7, 8])
    M, N, K = 5, 3, 7
    ar, ac = (M, K) if opA == "N" else (K, M)
    br, bc = (K, N) if opB == "N" else (N, K)
    A = np.broadcast_to(p, (ac, ar, 4)).copy()
    B = np.broadcast_to(q, (bc, br, 4)).copy()
    C = np.full((N, M, 4), np.nan)
    oracle.qgemm(opA, opB, M, N, K, 1, A, B, 0, C)
    expect = K * g[label][2]
    assert np.all(C == expect)


def test_identity_A_and_left_scalars():
    """P9 / A2: A = I => C = alpha op(B) + beta C, alpha and beta from the LEFT
    (P:493-500): alpha = e1, B = e2 gives e1 e2 = e3 (a right product would give
    -e3, basis table)."""
    e = np.eye(4)
    A = np.zeros((1, 1, 4)); A[0, 0] = e[0]
    B = np.zeros((1, 1, 4)); B[0, 0] = e[2]
    C = np.zeros((1, 1, 4)); C[0, 0] = e[3]
    oracle.qgemm("N", "N", 1, 1, 1, e[1], A, B, e[2], C)
    # e1*e2 + e2*e3 = e3 + e1
    np.testing.assert_array_equal(C[0, 0], e[3] + e[1])


def test_scalar_case():
    """M = N = K = 1 reduces to the scalar product."""
    g = _golden_products()
    A = g["pq"][0].reshape(1, 1, 4).copy()
    B = g["pq"][1].reshape(1, 1, 4).copy()
    C = np.full((1, 1, 4), np.nan)
    oracle.qgemm("N", "N", 1, 1, 1, 1, A, B, 0, C)
    np.testing.assert_array_equal(C[0, 0], g["pq"][2])


def test_alpha0_beta1_unchanged_and_beta0_nan_safe():
    """alpha = 0, beta = 1 leaves C bitwise unchanged; beta = 0 never reads C (R3)."""
    pr = make_problem(5, 6, 7, "N", "N", 0, 1, seed=3)
    C0 = pr.C.copy()
    oracle.qgemm("N", "N", 5, 6, 7, 0, pr.A, pr.B, 1, pr.C)
    np.testing.assert_array_equal(pr.C, C0)
    pr = make_problem(5, 6, 7, "N", "N", 1, 0, seed=3, c_init="nan")
    oracle.qgemm("N", "N", 5, 6, 7, 1, pr.A, pr.B, 0, pr.C)
    assert np.all(np.isfinite(pr.C[:, :5, :]))


def test_K0_is_beta_scale():
    """K = 0: C <- beta C (empty sum, R4)."""
    pr = make_problem(4, 3, 0, "N", "N", 1, (0, 1, 0, 0), seed=2)
    C0 = pr.C.copy()
    oracle.qgemm("N", "N", 4, 3, 0, 1, pr.A, pr.B, (0, 1, 0, 0), pr.C)
    ref = reference_gemm_via_chi("N", "N", 0, np.zeros((4, 0, 4)), np.zeros((0, 3, 4)),
                                 (0, 1, 0, 0), storage_to_logical(C0, 4))
    np.testing.assert_allclose(storage_to_logical(pr.C, 4), ref, atol=1e-15, rtol=0)


# ---------------------------------------------------------------- helpers of the oracle
@pytest.mark.parametrize("opA,opB", [("N", "N"), ("T", "H"), ("H", "T")])
def test_entries_equal_full(opA, opB):
    """qgemm_entries (sampled parity at full sizes) == qgemm bitwise (same
    summation order), pinned through the full oracle above."""
    M, N, K = 13, 11, 9
    pr = make_problem(M, N, K, opA, opB, (0.5, 0.1, -0.2, 0.3), (-1, 0, 0.5, 0), seed=4,
                      ldc=M + 1)
    C0 = pr.C.copy()
    oracle.qgemm(opA, opB, M, N, K, pr.alpha, pr.A, pr.B, pr.beta, pr.C)
    rows = np.array([0, 12, 5, 7, 3]); cols = np.array([0, 10, 3, 0, 9])
    ent = oracle.qgemm_entries(opA, opB, M, N, K, pr.alpha, pr.A, pr.B, pr.beta, C0, rows, cols)
    for s in range(rows.size):
        np.testing.assert_array_equal(ent[s], pr.C[cols[s], rows[s]])


@pytest.mark.parametrize("op", ["N", "T", "H"])
def test_qgemv_vs_complex(op):
    """qgemv (Freivalds helper) vs chi(op(X)) @ chi(x) with numpy."""
    rng = np.random.default_rng(12)
    r, c = 6, 5
    X = quat_matrix(rng, r if op == "N" else c, c if op == "N" else r, None)
    x = rng.standard_normal((c, 4))
    y = oracle.qgemv(op, r, c, X, x)
    LX = op_materialise(op, storage_to_logical(X, r if op == "N" else c))
    ref = unchi(chi(LX) @ chi(x.reshape(c, 1, 4)))
    np.testing.assert_allclose(y, ref[:, 0, :], atol=1e-14, rtol=0)


def test_thread_count_independent():
    """Every column is computed by one thread in one order: bitwise equal for 1 vs 4 threads."""
    pr = make_problem(33, 17, 29, "T", "N", 1, 0, seed=1)
    C1 = pr.C.copy(); C4 = pr.C.copy()
    oracle.qgemm("T", "N", 33, 17, 29, 1, pr.A, pr.B, 0, C1, nthreads=1)
    oracle.qgemm("T", "N", 33, 17, 29, 1, pr.A, pr.B, 0, C4, nthreads=4)
    np.testing.assert_array_equal(C1, C4)


def test_bad_op_rejected():
    pr = make_problem(2, 2, 2)
    with pytest.raises(ValueError):
        oracle.qgemm("X", "N", 2, 2, 2, 1, pr.A, pr.B, 0, pr.C)


def test_embedding_roundtrip():
    rng = np.random.default_rng(0)
    L = storage_to_logical(quat_matrix(rng, 5, 3), 5)
    np.testing.assert_array_equal(unchi(chi(L)), L)
    X = logical_to_storage(L, ld=7)
    np.testing.assert_array_equal(storage_to_logical(X, 5), L)


def test_counter_generator_torch_cpu_matches_numpy():
    """synth/gpu_gen.py (torch int64 ops) reproduces synth.inputs.counter_uniform bitwise."""
    import torch
    from synth.gpu_gen import counter_hermitian, counter_matrix, counter_uniform_t, host_rows_N
    from synth.inputs import counter_uniform
    idx = np.random.default_rng(0).integers(0, 1 << 40, 5000)
    np.testing.assert_array_equal(counter_uniform_t(3, 1, torch.from_numpy(idx)).numpy(),
                                  counter_uniform(3, 1, idx))
    M = counter_matrix(3, 1, 50, 40, "cpu").numpy()
    np.testing.assert_array_equal(M[:, [0, 7, 49], :], host_rows_N(3, 1, 50, [0, 7, 49], 40))
    H = counter_hermitian(5, 2, 30, "cpu", chunk_cols=7).numpy()
    L = H.transpose(1, 0, 2)
    LH = L.transpose(1, 0, 2).copy()
    LH[..., 1:] *= -1
    np.testing.assert_array_equal(L, LH)


def test_counter_block_generators():
    """synth: a row/column block of the global counter matrix (a rank's shard) is
    the slice of the whole matrix; torch and numpy twins agree (uniform bitwise,
    Box-Muller normal to rounding); the normal draws have N(0,1) moments; a row
    block of the Hermitian initialiser is the slice of the whole one."""
    import torch
    from synth.gpu_gen import counter_block, counter_hermitian, counter_matrix
    from synth.inputs import counter_block_host
    full = counter_matrix(4, 2, 50, 30, "cpu").numpy()
    blk = counter_block(4, 2, 50, 7, 20, 3, 11, "cpu", chunk_cols=4).numpy()
    np.testing.assert_array_equal(blk, full[3:14, 7:27, :])
    np.testing.assert_array_equal(blk, counter_block_host(4, 2, 50, 7, 20, 3, 11))
    zt = counter_block(1, 9, 300, 0, 300, 0, 200, "cpu", dist="normal").numpy()
    zh = counter_block_host(1, 9, 300, 0, 300, 0, 200, dist="normal")
    assert np.abs(zt - zh).max() <= 1e-14 * max(1.0, np.abs(zh).max())
    assert abs(zh.mean()) < 0.01 and abs(zh.var() - 1.0) < 0.01
    assert np.isfinite(zh).all()
    H = counter_hermitian(5, 2, 30, "cpu").numpy()
    Hr = counter_hermitian(5, 2, 30, "cpu", chunk_cols=4, r0=9, nrows=13).numpy()
    np.testing.assert_array_equal(Hr, H[:, 9:22, :])
    del torch
