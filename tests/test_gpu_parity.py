"""CUDA path (through the C ABI) vs the CPU oracle, element by element (-m gpu).

Tolerances are the north star's (tests/tolerance.py): FP64
1e-12 K max|A| max|B|, FP32 1e-4 sqrt(K) max|A| max|B| (+ reading R8).
Exact-integer inputs require bitwise equality.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
import paper_1903_05575_b200 as qg
from synth import CONFIGS, make_problem
from tests.gpu_helpers import assert_parity, oracle_full, path_policy, run_gpu, to_dev

pytestmark = pytest.mark.gpu
OPS = [(a, b) for a in "NTH" for b in "NTH"]
QALPHA = (0.3, -1.2, 0.7, 0.25)
QBETA = (-0.5, 0.1, -0.9, 0.4)
# pack launch + persistent mainloop | one-launch small kernel (tile-exact variant where
# the shape allows) | the small kernel's general variant only | TMA-fed mainloop (no
# pack): 4-quaternion-group tiles where the extents allow (else 32-byte tiles) | 32-byte
# tiles only
PATHS = [qg.PATH_PACKED, qg.PATH_SMALL, qg.PATH_SMALL_GENERAL, qg.PATH_DIRECT, qg.PATH_DIRECT32]


@pytest.fixture(params=PATHS, ids=["packed", "small", "small_general", "direct", "direct32"])
def path(request):
    with path_policy(request.param):
        yield request.param


def _lds(opA, opB, M, N, K, pad):
    lda = (M if opA == "N" else K) + pad
    ldb = (K if opB == "N" else N) + pad
    return lda, ldb, M + pad


# ---------------------------------------------------------------- config 1
def test_c1_full(path):
    cfg = CONFIGS["c1"]
    pr = make_problem(cfg["M"], cfg["N"], cfg["K"], "N", "N", cfg["alpha"], cfg["beta"], seed=0,
                      c_init="nan")
    assert_parity(pr, run_gpu(pr), oracle_full(pr))


# ---------------------------------------------------------------- config 2
@pytest.mark.parametrize("opA,opB", OPS)
def test_c2_all_ops_padded_ld(opA, opB):
    cfg = CONFIGS["c2"]
    n = cfg["M"]
    pr = make_problem(n, n, n, opA, opB, cfg["alpha"], cfg["beta"], seed=0, lda=cfg["ld"],
                      ldb=cfg["ld"], ldc=cfg["ld"])
    assert np.isnan(pr.A[:, n:, :]).all() and np.isnan(pr.B[:, n:, :]).all()
    assert_parity(pr, run_gpu(pr), oracle_full(pr))


# ---------------------------------------------------------------- ragged sweep
SIZES = [1, 2, 3, 5, 7, 8, 17, 33, 63, 64, 65, 127, 129]


@pytest.mark.parametrize("opA,opB", OPS)
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_ragged_shapes_quaternion_scalars(opA, opB, seed, path):
    rng = np.random.default_rng(100 + seed)
    for _ in range(4):
        M, N, K = (int(rng.choice(SIZES)) for _ in range(3))
        lda, ldb, ldc = _lds(opA, opB, M, N, K, int(rng.integers(0, 3)))
        pr = make_problem(M, N, K, opA, opB, QALPHA, QBETA, seed=seed, lda=lda, ldb=ldb, ldc=ldc)
        assert_parity(pr, run_gpu(pr), oracle_full(pr))


@pytest.mark.parametrize("M,N,K", [(200, 130, 300), (64, 64, 16), (65, 191, 33), (1, 300, 257)])
@pytest.mark.parametrize("opA,opB", OPS)
def test_exact_integer_bitwise_f64(M, N, K, opA, opB, path):
    """P8: integer components in [-8, 8] -> exact in any order -> bitwise."""
    pr = make_problem(M, N, K, opA, opB, (2, -1, 0, 3), (1, 0, -2, 1), seed=3, dist="int8")
    assert_parity(pr, run_gpu(pr), oracle_full(pr), exact=True)


@pytest.mark.parametrize("M,N,K,pad", [(196, 132, 84, 3), (4, 8, 4, 1), (260, 68, 1028, 2),
                                       (64, 128, 16, 0), (132, 36, 37, 1)])
@pytest.mark.parametrize("opA,opB", OPS)
def test_group4_tma_feed(M, N, K, pad, opA, opB):
    """Direct path with whole 4-quaternion groups (M, N, K multiples of 4; the last
    shape's K = 37 keeps the 32-byte feed whenever an operand is k-contiguous), so
    the 128-byte-swizzle group tiles with the permuted k order run: tile-ragged
    edges, odd ld padding (NaN), stream-K splits, quaternion alpha/beta;
    exact-integer inputs -> bitwise."""
    lda, ldb, ldc = _lds(opA, opB, M, N, K, pad)
    with path_policy(qg.PATH_DIRECT):
        pr = make_problem(M, N, K, opA, opB, QALPHA, QBETA, seed=7, lda=lda, ldb=ldb, ldc=ldc)
        assert_parity(pr, run_gpu(pr), oracle_full(pr))
        pr = make_problem(M, N, K, opA, opB, (2, -1, 0, 3), (1, 0, -2, 1), seed=8, dist="int8",
                          lda=lda, ldb=ldb, ldc=ldc)
        assert_parity(pr, run_gpu(pr), oracle_full(pr), exact=True)


@pytest.mark.parametrize("M,N,K", [(300, 260, 700), (512, 512, 64), (1000, 130, 4000), (257, 129, 33)])
@pytest.mark.parametrize("opA,opB", [("N", "H"), ("T", "N"), ("H", "T")])
@pytest.mark.parametrize("policy", [qg.PATH_PACKED, qg.PATH_DIRECT], ids=["packed", "direct"])
def test_f32_split_k_pair_kernel(M, N, K, opA, opB, policy):
    """FP32 tcgen05 pair kernel with fewer tile pairs than a wave: K split over
    up to 8 clusters per tile pair, raw partials summed by the reduce + epilogue
    launch (1000 x 130 x 4000: several accumulation chunks per split).  Packed
    chunks, and the direct feed (raw tiles by TMA, hi/lo split by the converter
    warps).  Tolerance on normal inputs; bitwise on exact-integer inputs."""
    with path_policy(policy):
        pr = make_problem(M, N, K, opA, opB, QALPHA, QBETA, seed=13, dist="normal")
        assert_parity(pr, run_gpu(pr, "f32"), oracle_full(pr), precision="f32")
        pr = make_problem(M, N, K, opA, opB, (1, 0, 0, 0), (-1, 0, 0, 0), seed=14, dist="int2")
        assert_parity(pr, run_gpu(pr, "f32"), oracle_full(pr), exact=True)


@pytest.mark.parametrize("M,N,K,S", [(2048, 2048, 1024, 4), (2000, 1900, 777, 3)])
@pytest.mark.parametrize("opA,opB", [("N", "H"), ("H", "T")])
def test_f32_remainder_split_above_one_wave(M, N, K, S, opA, opB):
    """FP32 pair kernel above one wave of 74 tile pairs: the whole waves run whole
    pairs, the pairs of the partial last wave split K: 2048^2 has
    128 pairs = 74 + 54 whole + 54 x 4 quarter-K units; 2000 x 1900 has 120 =
    74 + 46 x 3 (ragged M / N tiles and a K of 98 k-tiles split 32/33/33).  Both
    feeds; normal inputs within the FP32 tolerance, exact-integer inputs
    bitwise; the launch count shows the reduce launch ran (split taken)."""
    prs = [make_problem(M, N, K, opA, opB, QALPHA, QBETA, seed=21, dist="normal"),
           make_problem(M, N, K, opA, opB, (1, 0, 0, 0), (-1, 0, 0, 0), seed=22, dist="int2")]
    refs = [oracle_full(pr) for pr in prs]
    for policy, launches in ((qg.PATH_PACKED, 3), (qg.PATH_DIRECT, 2)):
        with path_policy(policy):
            for pr, ref, exact in zip(prs, refs, (False, True)):
                got = run_gpu(pr, "f32")
                assert qg.last_launch_count() == launches, (policy, S)
                assert_parity(pr, got, ref, precision="f32", exact=exact)


@pytest.mark.parametrize("M,N,K", [(1024, 1024, 16), (1024, 1024, 48), (1000, 1030, 20), (2048, 640, 64)])
@pytest.mark.parametrize("opA,opB", [("N", "H"), ("T", "N")])
def test_ring_epilogue_short_k_stream_k(M, N, K, opA, opB):
    """The ring epilogue at every K (store warp): 1-4 k-tiles per
    tile, more tiles than one wave, so whole tiles, stream-K owners (ring
    epilogue after the fixup) and contributors (no C stages) interleave in each
    CTA's work list and the store warp must track the producer's slot sequence
    exactly; ragged tiles; beta != 0 (the ring) with quaternion alpha/beta, and
    beta = 0 (per-lane stores); exact-integer inputs -> bitwise."""
    with path_policy(qg.PATH_DIRECT):
        for beta in (QBETA, (0, 0, 0, 0)):
            pr = make_problem(M, N, K, opA, opB, QALPHA, beta, seed=31, ldc=M + 1)
            assert_parity(pr, run_gpu(pr), oracle_full(pr))
        pr = make_problem(M, N, K, opA, opB, (2, -1, 0, 3), (1, 0, -2, 1), seed=32, dist="int8")
        assert_parity(pr, run_gpu(pr), oracle_full(pr), exact=True)


@pytest.mark.parametrize("M,N,K", [(1024, 1024, 48), (300, 260, 700), (130, 70, 520), (1, 64, 600)])
@pytest.mark.parametrize("opA,opB", [("N", "H"), ("T", "N"), ("H", "H")])
@pytest.mark.parametrize("alpha", [(1, 0, 0, 0), (0.75, 0, 0, 0), QALPHA], ids=["a1", "areal", "aquat"])
def test_ring_epilogue_beta_one_tma_reduction(M, N, K, opA, opB, alpha):
    """beta == 1 (c3, c4, QHERK's configs): the ring epilogue writes alpha (x) acc
    and the store warp adds each box into C with a TMA reduction,
    no C read through shared memory; ragged tiles, padded ldc (the sentinel in
    C's padding must survive the reduction), stream-K owners; real and
    quaternion alpha; exact-integer inputs -> bitwise."""
    with path_policy(qg.PATH_DIRECT):
        pr = make_problem(M, N, K, opA, opB, alpha, (1, 0, 0, 0), seed=41, ldc=M + 3)
        assert_parity(pr, run_gpu(pr), oracle_full(pr))
        ia = tuple(int(round(2 * x)) for x in alpha)
        pr = make_problem(M, N, K, opA, opB, ia, (1, 0, 0, 0), seed=42, dist="int8", ldc=M + 3)
        assert_parity(pr, run_gpu(pr), oracle_full(pr), exact=True)


@pytest.mark.parametrize("M,N,K", [(1024, 1024, 48), (300, 260, 700), (130, 70, 520), (1, 64, 600)])
@pytest.mark.parametrize("opA,opB", [("N", "N"), ("T", "H")])
def test_ring_epilogue_beta_zero_nan_c(M, N, K, opA, opB):
    """beta == 0 (c5's config) through the ring epilogue (QG_RING_BETA0): no C
    stage is loaded, the store warp TMA-stores alpha (x) acc; a NaN-filled C must
    not leak into the result (beta = 0 means C is not read), ragged
    tiles, stream-K owners; exact-integer inputs -> bitwise."""
    with path_policy(qg.PATH_DIRECT):
        pr = make_problem(M, N, K, opA, opB, QALPHA, 0, seed=43, c_init="nan")
        assert_parity(pr, run_gpu(pr), oracle_full(pr))
        pr = make_problem(M, N, K, opA, opB, (2, -1, 0, 3), 0, seed=44, dist="int8", c_init="nan")
        assert_parity(pr, run_gpu(pr), oracle_full(pr), exact=True)


@pytest.mark.parametrize("M,N,K", [(130, 70, 520), (64, 1, 512), (1, 64, 600), (257, 129, 1000)])
@pytest.mark.parametrize("opA,opB", OPS)
@pytest.mark.parametrize("policy", [qg.PATH_PACKED, qg.PATH_DIRECT], ids=["packed", "direct"])
def test_ring_epilogue_edges(M, N, K, opA, opB, policy):
    """K >= 512 (>= 32 k-tiles; since the store warp the ring applies at every K,
    see test_ring_epilogue_short_k_stream_k): the FP64 epilogue reads C through the ring (TMA
    load, update in shared memory, TMA store clipped at the M / N edges), on
    ragged tiles, degenerate M or N, padded ld (sentinel in C's padding must
    survive), quaternion alpha/beta; exact-integer inputs -> bitwise."""
    with path_policy(policy):
        pr = make_problem(M, N, K, opA, opB, QALPHA, QBETA, seed=15, ldc=M + 3)
        assert_parity(pr, run_gpu(pr), oracle_full(pr))
        pr = make_problem(M, N, K, opA, opB, (2, -1, 0, 3), (1, 0, -2, 1), seed=16, dist="int8",
                          ldc=M + 3)
        assert_parity(pr, run_gpu(pr), oracle_full(pr), exact=True)


@pytest.mark.parametrize("opA,opB", OPS)
def test_exact_integer_bitwise_f32(opA, opB, path):
    """P8 in FP32: |partial sums| <= 2^24, so FP32 is exact too."""
    pr = make_problem(150, 70, 200, opA, opB, (1, 0, 0, 0), (-1, 0, 0, 0), seed=4, dist="int8")
    assert_parity(pr, run_gpu(pr, "f32"), oracle_full(pr), exact=True)


@pytest.mark.parametrize("opA,opB", OPS)
def test_f32_tolerance(opA, opB, path):
    """FP32 variant checked against the FP64 oracle on the FP64 inputs (R11)."""
    pr = make_problem(257, 190, 513, opA, opB, QALPHA, QBETA, seed=5, dist="normal",
                      lda=(257 if opA == "N" else 513) + 1)
    assert_parity(pr, run_gpu(pr, "f32"), oracle_full(pr), precision="f32")


# ---------------------------------------------------------------- K-panel loop (a6)
@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_k_panel_loop_small_workspace(precision):
    """Workspace for 3 K-tiles only: the call loops over K-panels, beta on the
    first, accumulate afterwards (Alg. 2 kappa loop)."""
    M, N, K = 130, 100, 16 * 7 + 5
    pr = make_problem(M, N, K, "H", "T", QALPHA, QBETA, seed=6)
    dt = torch.float64 if precision == "f64" else torch.float32
    with path_policy(qg.PATH_PACKED):
        full = qg.workspace_bytes("H", "T", M, N, K, dt)
        mn = qg.workspace_min_bytes("H", "T", M, N, K, dt)
    kt = (K + 15) // 16
    per_ktile = (full - mn) // (kt - 1)
    small = mn + 2 * per_ktile  # room for 3 K-tiles -> panels of 3, 3, 2
    assert small < full
    ws = torch.empty(small, dtype=torch.uint8, device="cuda")
    with path_policy(qg.PATH_PACKED):
        got = run_gpu(pr, precision, workspace=ws)
    assert qg.last_launch_count() == 3 * 2  # 3 panels x (pack A+B, mainloop)
    assert_parity(pr, got, oracle_full(pr), precision=precision)


# ---------------------------------------------------------------- degenerate cases
def test_quick_returns_and_beta_paths(path):
    # M = 0 / N = 0: nothing enqueued, C untouched
    pr = make_problem(5, 4, 3, seed=1)
    C = to_dev(pr.C)
    C0 = C.clone()
    A, B = to_dev(pr.A), to_dev(pr.B)
    qg.qgemm("N", "N", 1, A, B, 1, C, M=0, N=4, K=3)
    assert qg.last_launch_count() == 0
    qg.qgemm("N", "N", 1, A, B, 1, C, M=5, N=0, K=3)
    assert torch.equal(C, C0)
    # alpha = 0, beta = 1 -> bitwise unchanged, nothing enqueued
    qg.qgemm("N", "N", 0, A, B, 1, C, M=5, N=4, K=3)
    assert qg.last_launch_count() == 0
    torch.cuda.synchronize()
    assert torch.equal(C, C0)
    # K = 0 -> beta C (quaternion beta, left)
    pr = make_problem(6, 5, 0, "N", "N", 1, QBETA, seed=2)
    assert_parity(pr, run_gpu(pr), oracle_full(pr))
    # beta = 0 with NaN C -> finite
    pr = make_problem(70, 33, 20, "T", "H", QALPHA, 0, seed=2, c_init="nan")
    got = run_gpu(pr)
    assert np.isfinite(got[:, :70]).all()
    assert_parity(pr, got, oracle_full(pr))


def test_alias_rejected_and_nothing_enqueued():
    pr = make_problem(8, 8, 8, seed=0)
    A = to_dev(pr.A)
    with pytest.raises(qg.QgemmError) as ei:
        qg.qgemm("N", "N", 1, A, A, 0, A)
    assert ei.value.code == -12


def test_naive_cross_check_and_stream(path):
    """Debug kernel and tuned kernel agree on a side stream."""
    pr = make_problem(190, 77, 140, "H", "N", QALPHA, QBETA, seed=9)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        got = run_gpu(pr, stream=s)
        nai = run_gpu(pr, naive=True, stream=s)
    ref = oracle_full(pr)
    assert_parity(pr, got, ref)
    assert_parity(pr, nai, ref)


def test_b_is_a_hermitian_rank_k_shape(path):
    """c4's structure at reduced M: C <- A A^H + C with B == A (same buffer) and a
    Hermitian C; the result is Hermitian (P12) and matches the oracle."""
    n, K = 320, 256
    pr = make_problem(n, n, K, "N", "H", 1, 1, seed=0, c_init="hermitian", b_is_a=True)
    got = run_gpu(pr)
    assert_parity(pr, got, oracle_full(pr))
    L = got[:, :n, :].transpose(1, 0, 2)
    LH = L.transpose(1, 0, 2).copy(); LH[..., 1:] *= -1
    assert np.abs(L - LH).max() <= 1e-12 * K


# ---------------------------------------------------------------- config 3 at full size
@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_c3_full_size_sampled_and_freivalds(precision):
    """c3 (8192^3, N/H, alpha = beta = 1, N(0,1)) in the bench's launch
    configuration:
      * 16 full rows (every 512th row) and 2 full columns of C from the oracle,
        entry by entry within the per-entry tolerance;
      * a block Freivalds check of the WHOLE C (tests/freivalds.py: right vectors
        supported on column blocks of 64 (FP64) / 4 (FP32) columns), passing
        below a bound calibrated on the 16 known rows (20 x (FP64) / 3 x (FP32)
        the largest residual there), which must itself be small enough that any
        single entry off by 10 x tol is caught (freivalds.detects).  FP32: the
        tcgen05 accumulation (truncating FP32 adds over ~12k MMA steps per output)
        leaves per-entry errors of a few percent of tol, so its blocks are short
        and its factor small;
      * negative control: the same check on C with ONE unsampled entry moved by
        10 x tol must fail."""
    from tests.freivalds import Check, columns_of, detects, draw_x, qnorm, times_x
    from tests.gpu_helpers import tol_for
    cfg = CONFIGS["c3"]
    n = cfg["M"]
    pr = make_problem(n, n, n, "N", "H", cfg["alpha"], cfg["beta"], seed=0, dist="normal")
    got = run_gpu(pr, precision)                      # (n, n, 4): columns of C
    tol = tol_for(pr, precision)
    rows = np.arange(0, n, 512) + 17                  # 16 full rows
    A_S = np.ascontiguousarray(pr.A[:, rows, :])      # op(A) rows S (stored (K, |S|, 4))
    ref_rows = np.ascontiguousarray(pr.C[:, rows, :])
    oracle.qgemm("N", "H", rows.size, n, n, pr.alpha, A_S, pr.B, pr.beta, ref_rows)
    got_rows = np.ascontiguousarray(got[:, rows, :])
    err_rows = float(np.abs(got_rows - ref_rows).max())
    assert err_rows <= tol, (err_rows, tol)
    cols = np.array([5, n - 2])
    ref_cols = np.ascontiguousarray(pr.C[cols])
    B_cols = np.ascontiguousarray(pr.B[:, cols, :])   # op(B) = B^H: columns = rows of stored B
    oracle.qgemm("N", "H", n, cols.size, n, pr.alpha, pr.A, B_cols, pr.beta, ref_cols)
    err_cols = float(np.abs(got[cols] - ref_cols).max())
    assert err_cols <= tol, (err_cols, tol)
    # block Freivalds over the whole C
    bs, factor = (64, 20.0) if precision == "f64" else (4, 3.0)
    x = draw_x(n, seed=7)
    Y = times_x(lambda j0, j1: (pr.B[:, j0:j1, :], "H"), n, n, x, bs)   # op(B) X: (nb, K, 4)
    AY = np.zeros((Y.shape[0], n, 4))
    oracle.qgemm("N", "N", n, Y.shape[0], n, 1, pr.A, Y, 0, AY)
    C0X = times_x(columns_of(pr.C), n, n, x, bs)
    chk = Check(n, n, bs, x, AY + C0X)                # alpha = beta = 1
    bound = chk.bound(ref_rows, got_rows, rows, factor)
    assert detects(bound, tol, factor), (bound, tol)  # power: 10 x tol on one entry is visible
    res = float(qnorm(chk.residual(columns_of(got))).max())
    assert res <= bound, (res, bound, tol)
    # negative control: one entry (row not sampled, column not sampled) moved by 10 tol
    bad = got.copy()
    bad[4321, 2345, 0] += 10 * tol
    res_bad = float(qnorm(chk.residual(columns_of(bad))).max())
    assert res_bad > bound, (res_bad, bound, tol)


# ---------------------------------------------------------------- small-problem path
def test_auto_policy_picks_one_launch_for_small_shapes():
    """c1 under the default policy: one kernel, no workspace (NEXT item 4)."""
    cfg = CONFIGS["c1"]
    assert qg.workspace_bytes("N", "N", 64, 64, 64) == 0
    pr = make_problem(cfg["M"], cfg["N"], cfg["K"], "N", "N", cfg["alpha"], cfg["beta"], seed=1)
    got = run_gpu(pr)
    assert qg.last_launch_count() == 1
    assert_parity(pr, got, oracle_full(pr))
    assert qg.workspace_bytes("N", "N", 1024, 1024, 1024) > 0  # c2 stays on the packed path


@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (8, 8, 4), (9, 7, 3), (40, 3, 1000), (3, 700, 9),
                                   (256, 256, 256), (31, 257, 64), (4000, 2, 5), (64, 64, 4096),
                                   (16, 24, 2053), (8, 8, 100), (5, 3, 2001)])
@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_small_kernel_split_and_edges(M, N, K, precision):
    """Every split factor S (1/2/4 warps per 8x8 tile over K) and cluster split Z
    (1..8 CTAs per tile over K, partials through distributed shared memory),
    ragged M/N/K tails, long-K and skinny shapes, both storage types, through
    the small path."""
    pr = make_problem(M, N, K, "T", "H", QALPHA, QBETA, seed=11, dist="normal",
                      lda=K + 1, ldb=N + 2, ldc=M + 3)
    with path_policy(qg.PATH_SMALL):
        got = run_gpu(pr, precision)
        assert qg.last_launch_count() == 1
    assert_parity(pr, got, oracle_full(pr), precision=precision)


@pytest.mark.parametrize("opA,opB", OPS)
def test_small_kernel_cluster_split_exact(opA, opB):
    """Cluster split over K (Z = 8: 64 tiles x 8 CTAs) with exact-integer inputs:
    the DSMEM reduction must give the oracle's result bitwise, for every op pair."""
    pr = make_problem(64, 56, 3001, opA, opB, (2, -1, 0, 3), (1, 0, -2, 1), seed=12, dist="int8")
    with path_policy(qg.PATH_SMALL):
        got = run_gpu(pr)
    assert_parity(pr, got, oracle_full(pr), exact=True)


@pytest.mark.parametrize("opA,opB", OPS)
@pytest.mark.parametrize("precision", ["f64", "f32"])
@pytest.mark.parametrize("M,N,K", [(64, 64, 64), (8, 8, 4), (40, 24, 12), (128, 64, 256), (16, 8, 1024)])
def test_tiny_kernel_exact_every_op_pair(opA, opB, precision, M, N, K):
    """The tile-exact small kernel (M % 8 == N % 8 == K % 4 == 0: c1's shape and
    its neighbours; op pair and conj signs compiled in, 256-bit quaternion
    accesses): bitwise equal to the oracle with exact-integer inputs and
    quaternion alpha/beta, for every op pair, in both storage precisions --
    and bitwise equal to the general small kernel (policy 5) on the same call.
    (40 x 24: the last CTA row holds tiles past M; 16 x 8 x 1024: K split over
    the warps of a CTA.)"""
    pr = make_problem(M, N, K, opA, opB, (2, -1, 0, 1), (1, 0, -1, 2), seed=M + N + K, dist="int2")
    with path_policy(qg.PATH_SMALL):
        got = run_gpu(pr, precision)
        assert qg.last_launch_count() == 1
    with path_policy(qg.PATH_SMALL_GENERAL):
        gen = run_gpu(pr, precision)
    assert_parity(pr, got, oracle_full(pr), exact=True)
    np.testing.assert_array_equal(got, gen)


def test_tiny_kernel_misaligned_base_takes_general_kernel():
    """An FP64 operand 16 but not 32 bytes aligned cannot take the tile-exact
    kernel's 256-bit accesses: the call falls back to the general small kernel
    (same result, bitwise with exact-integer inputs)."""
    pr = make_problem(64, 64, 64, "N", "N", 1, 0, seed=3, dist="int8")
    A = torch.empty(pr.A.size + 2, dtype=torch.float64, device="cuda")[2:].view(pr.A.shape)
    A.copy_(torch.from_numpy(pr.A))
    assert A.data_ptr() % 32 == 16
    B, C = to_dev(pr.B), to_dev(pr.C)
    with path_policy(qg.PATH_SMALL):
        qg.qgemm("N", "N", 1.0, A, B, 0.0, C)
    torch.cuda.synchronize()
    assert_parity(pr, C.cpu().numpy(), oracle_full(pr), exact=True)


def test_concurrent_streams_do_not_share_workspace():
    """Two calls in flight on two streams with library-managed workspaces: each
    stream gets its own scratch (a shared one would let the second call's pack
    overwrite the first call's packed operands)."""
    prs = [make_problem(700, 650, 900, "N", "H", QALPHA, QBETA, seed=30 + i) for i in range(2)]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = []
    for pr, s in zip(prs, streams):
        A, B, C = to_dev(pr.A), to_dev(pr.B), to_dev(pr.C)
        torch.cuda.synchronize()
        with torch.cuda.stream(s):
            qg.qgemm(pr.transA, pr.transB, pr.alpha, A, B, pr.beta, C, M=pr.M, N=pr.N, K=pr.K)
        outs.append((A, B, C))
    torch.cuda.synchronize()
    ws = {id(qg.get_workspace(1, "cuda", s)) for s in streams}
    assert len(ws) == 2
    for pr, (_, _, C) in zip(prs, outs):
        assert_parity(pr, C.cpu().numpy(), oracle_full(pr))


# ---------------------------------------------------------------- randomized sweep
def _random_cases(n, seed=2026):
    rng = np.random.default_rng(seed)
    sizes = [1, 3, 8, 16, 31, 64, 65, 100, 128, 129, 200, 257, 300, 513]
    for _ in range(n):
        M, N, K = (int(rng.choice(sizes)) for _ in range(3))
        opA, opB = str(rng.choice(list("NTH"))), str(rng.choice(list("NTH")))
        pads = rng.integers(0, 4, 3)
        alpha = tuple(rng.uniform(-1, 1, 4)) if rng.random() < 0.5 else (float(rng.uniform(-2, 2)),)
        beta = (0.0,) if rng.random() < 0.2 else tuple(rng.uniform(-1, 1, 4))
        yield M, N, K, opA, opB, pads, alpha, beta


@pytest.mark.parametrize("case", list(_random_cases(24)))
@pytest.mark.parametrize("precision", ["f64", "f32"])
def test_randomized_shapes_ops_scalars(case, precision, path):
    """Random shapes (ragged, skinny, K = 1), op pairs, ld padding, real or
    quaternion alpha and beta (beta = 0 with a NaN C) under every path policy."""
    M, N, K, opA, opB, pads, alpha, beta = case
    lda = (M if opA == "N" else K) + int(pads[0])
    ldb = (K if opB == "N" else N) + int(pads[1])
    pr = make_problem(M, N, K, opA, opB, alpha, beta, seed=M * 7 + N * 3 + K, dist="normal",
                      lda=lda, ldb=ldb, ldc=M + int(pads[2]),
                      c_init="nan" if beta == (0.0,) else "random")
    assert_parity(pr, run_gpu(pr, precision), oracle_full(pr), precision=precision)


_CONCURRENT = r"""
import sys, torch
sys.path.insert(0, {root!r})
import paper_1903_05575_b200 as qg
torch.manual_seed(0)
n = 1024  # 256 tiles on 148 SMs: an all-stream-K schedule (owners wait for contributors)
streams = [torch.cuda.Stream() for _ in range(3)]
ops = [("N", "N"), ("T", "H"), ("H", "N")]
data = []
for (oa, ob), s in zip(ops, streams):
    A = torch.randn(n, n, 4, dtype=torch.float64, device="cuda")
    B = torch.randn(n, n, 4, dtype=torch.float64, device="cuda")
    C0 = torch.randn(n, n, 4, dtype=torch.float64, device="cuda")
    data.append((oa, ob, A, B, C0, torch.empty_like(C0), s))
torch.cuda.synchronize()
ref = []
for oa, ob, A, B, C0, C, s in data:  # serial reference run (beta != 0: C goes through the ring)
    C.copy_(C0)
    qg.qgemm(oa, ob, 1.0, A, B, 0.5, C)
    ref.append(C.clone())
torch.cuda.synchronize()
for it in range(20):  # the three persistent grids in flight together
    for oa, ob, A, B, C0, C, s in data:
        with torch.cuda.stream(s):
            C.copy_(C0)
            qg.qgemm(oa, ob, 1.0, A, B, 0.5, C)
torch.cuda.synchronize()
for (oa, ob, A, B, C0, C, s), r in zip(data, ref):
    assert torch.equal(C, r), (oa, ob)  # same tile config -> bitwise
print("OK")
"""


def test_concurrent_persistent_grids_no_deadlock():
    """Three stream-K grids that each want every SM, in flight at once on three
    streams: the cooperative launch keeps each grid co-resident, so stream-K
    owners never wait for a contributor that cannot be scheduled (run in a
    subprocess with a timeout so a regression fails instead of hanging)."""
    import subprocess
    import sys as _sys
    root = __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__)))
    res = subprocess.run([_sys.executable, "-c", _CONCURRENT.format(root=root)], capture_output=True, text=True,
                         timeout=180)
    assert res.returncode == 0 and "OK" in res.stdout, res.stdout + res.stderr[-3000:]


@pytest.mark.parametrize("M,N,K,opA,opB", [(64, 64, 64, "N", "N"), (700, 650, 900, "N", "H"),
                                           (1024, 1024, 1024, "T", "N"), (300, 200, 100, "H", "T")])
def test_cuda_graph_capture_and_replay(M, N, K, opA, opB, path):
    """Every path (small kernel, pack + persistent mainloop with its flag memset
    and cooperative stream-K launch, TMA-fed direct) can be captured once and
    replayed: the replays reproduce the eager result bitwise."""
    pr = make_problem(M, N, K, opA, opB, QALPHA, 0.0, seed=40, c_init="zero")
    A, B = to_dev(pr.A), to_dev(pr.B)
    C_eager, C_graph = to_dev(pr.C), to_dev(pr.C)
    ws = torch.empty(max(256, qg.workspace_bytes(opA, opB, M, N, K)), dtype=torch.uint8, device="cuda")
    qg.qgemm(opA, opB, QALPHA, A, B, 0.0, C_eager, M=M, N=N, K=K, workspace=ws)
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        qg.qgemm(opA, opB, QALPHA, A, B, 0.0, C_graph, M=M, N=N, K=K, workspace=ws, stream=s)
    for _ in range(3):
        C_graph.fill_(float("nan"))
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(C_graph, C_eager)
    assert_parity(pr, C_eager.cpu().numpy(), oracle_full(pr))


@pytest.mark.parametrize("n", [2048, 4096])
def test_metamorphic_conjugate_transpose_identity(n):
    """(AB)^H = B^H A^H, checked on the GPU alone at sizes
    the oracle would take minutes for: qgemm('N','N', A, B) vs qgemm('H','H', B, A)."""
    g = torch.Generator(device="cuda").manual_seed(n)
    A = torch.randn((n, n, 4), dtype=torch.float64, device="cuda", generator=g)
    B = torch.randn((n, n, 4), dtype=torch.float64, device="cuda", generator=g)
    C1 = torch.zeros((n, n, 4), dtype=torch.float64, device="cuda")
    C2 = torch.zeros_like(C1)
    qg.qgemm("N", "N", 1.0, A, B, 0.0, C1)
    qg.qgemm("H", "H", 1.0, B, A, 0.0, C2)
    torch.cuda.synchronize()
    conjT = C1.transpose(0, 1) * torch.tensor([1.0, -1.0, -1.0, -1.0], dtype=torch.float64, device="cuda")
    tol = 2e-12 * n * float(A.abs().max()) * float(B.abs().max())
    assert float((C2 - conjT).abs().max()) <= tol


def test_f32_long_k_error_bounded_by_accumulation_chunks():
    """FP32 on the tensor cores: the TMEM accumulator adds truncate, so one
    accumulation chain's error grows like K^1.5 (tools/f32_accuracy.py) while
    the north-star tolerance grows like sqrt(K); the pair kernel therefore
    accumulates in chunks of 256 k and adds the chunks with round-to-nearest FP32
    (qg_tc32_2cta.cuh), which keeps the error a constant fraction of the
    tolerance (~0.2 for uniform data).  M = N = 2048, K = 32768 (128 tile pairs,
    no split-K; one 32768-deep chain gave ~7 x tol): max error / tol <= 0.5 on 2
    full rows and 2 full columns against the oracle on the FP64 inputs (R11)."""
    from synth.gpu_gen import counter_matrix, host_cols, host_rows_N
    n, K = 2048, 32768
    A = counter_matrix(0, 1, n, K, "cuda")             # stored n x K (op N)
    B = counter_matrix(0, 2, K, n, "cuda")             # stored K x n (op N)
    C = torch.zeros((n, n, 4), dtype=torch.float32, device="cuda")
    qg.qgemm_f32("N", "N", 1.0, A.float(), B.float(), 0.0, C)
    torch.cuda.synchronize()
    rows, cols = np.array([1, n - 3]), np.array([0, n - 1])
    A_S = host_rows_N(0, 1, n, rows, K)                # (K, 2, 4)
    B_C = host_cols(0, 2, K, cols, K)                  # (2, K, 4)
    B_h = counter_matrix(0, 2, K, n, "cpu").numpy()    # (n, K, 4)
    ref_r = np.zeros((n, rows.size, 4))
    oracle.qgemm("N", "N", rows.size, n, K, 1, A_S, B_h, 0, ref_r)
    A_h = counter_matrix(0, 1, n, K, "cpu").numpy()    # (K, n, 4)
    ref_c = np.zeros((cols.size, n, 4))
    oracle.qgemm("N", "N", n, cols.size, K, 1, A_h, B_C, 0, ref_c)
    got = C.double().cpu().numpy()
    err = max(float(np.abs(got[:, rows, :] - ref_r).max()), float(np.abs(got[cols] - ref_c).max()))
    tol = 1e-4 * K ** 0.5 * float(np.abs(A_h).max()) * float(np.abs(B_h).max())
    assert err <= 0.5 * tol, (err, tol)


def test_remote_c_epilogue_in_child_process():
    """The multi-GPU epilogue -- C in another GPU's memory (dist.qgemm_rowsharded_p2p
    stores row blocks into root's C over peer memory): per-lane loads / stores, no
    ring, no L2 prefetch of C.  On a one-GPU box every C is local, so the child
    process sets QG_FORCE_REMOTE_C=1 (read once by the library) and reruns the
    ring tests (beta = 1, beta = 0 with a NaN C, quaternion beta at short K with
    stream-K owners) and the exact-integer QHERK tests on that epilogue against
    the oracle."""
    import os
    import subprocess
    import sys as _sys
    if os.environ.get("QG_FORCE_REMOTE_C"):
        pytest.skip("already the child")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, QG_FORCE_REMOTE_C="1")
    cmd = [_sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
           "tests/test_gpu_parity.py", "tests/test_gpu_qherk.py",
           "-k", "ring_epilogue or qherk_exact_integer or qherk_multi_band"]
    res = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert res.returncode == 0 and " passed" in res.stdout, res.stdout[-3000:] + res.stderr[-3000:]
