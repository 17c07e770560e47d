"""qgemm_host / qgemm_host_f32 (host-resident operands streamed through device
staging, include/qgemm.h) vs the CPU oracle, element by element (-m gpu).

Shapes are chosen so the K-chunk loop has several chunks (Q > 2: staging
double buffer reused) and C several column panels (P > 1), with ragged tails
and ld padding (NaN in A/B padding, sentinel in C padding must survive)."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_1903_05575_b200 as qg
from synth import make_problem
from tests.gpu_helpers import assert_parity, oracle_full, path_policy

pytestmark = pytest.mark.gpu
OPS = [(a, b) for a in "NTH" for b in "NTH"]
QALPHA = (0.3, -1.2, 0.7, 0.25)
QBETA = (-0.5, 0.1, -0.9, 0.4)


def run_host(pr, precision="f64", pin=True, stream=None, workspace=None):
    dt = torch.float64 if precision == "f64" else torch.float32

    def host(x):
        t = torch.from_numpy(np.array(x, copy=True)).to(dt)  # never alias the problem's arrays
        return t.pin_memory() if pin else t

    A = host(pr.A)
    B = A if pr.B is pr.A else host(pr.B)
    C = host(pr.C)
    qg.qgemm_host(pr.transA, pr.transB, pr.alpha, A, B, pr.beta, C, M=pr.M, N=pr.N, K=pr.K,
                  stream=stream, workspace=workspace)
    (stream or torch.cuda.current_stream()).synchronize()
    return C.double().numpy()


@pytest.mark.parametrize("policy", [qg.PATH_AUTO, qg.PATH_PACKED], ids=["auto_direct", "packed"])
@pytest.mark.parametrize("opA,opB", OPS)
def test_host_chunked_all_ops(opA, opB, policy):
    M, N, K = 300, 520, 700  # K chunks 64/256/380 (growing x2), C panels 256/256/8
    lda = (M if opA == "N" else K) + 3
    ldb = (K if opB == "N" else N) + 1
    pr = make_problem(M, N, K, opA, opB, QALPHA, QBETA, seed=21, lda=lda, ldb=ldb, ldc=M + 2)
    with path_policy(policy):
        assert_parity(pr, run_host(pr), oracle_full(pr))
        # [3 packs (A+B per chunk), packed only] + 2 full mainloops + 1 beta*C
        # fold-in + 3 panel mainloops; auto reads the staged chunks in place (TMA)
        packs = 3 if policy == qg.PATH_PACKED else 0
        assert qg.last_launch_count() == packs + 2 + 1 + 3


@pytest.mark.parametrize("precision", ["f64", "f32"])
@pytest.mark.parametrize("opA,opB", [("N", "H"), ("T", "N")])
def test_host_big_last_chunk_and_split_last_panel(opA, opB, precision):
    """K = 1100 -> chunks 64/256/512/268, reordered so the longest runs last
    (64/256/268/512); N = 1024 -> 4 column panels of 256, the last one cut in
    two 128-column pieces (packed FP32 B panels start on 128-column tiles)."""
    pr = make_problem(256, 1024, 1100, opA, opB, QALPHA, QBETA, seed=24,
                      dist="normal" if precision == "f32" else "uniform")
    got = run_host(pr, precision)
    assert_parity(pr, got, oracle_full(pr), precision=precision)
    if precision == "f64":  # direct chunks: 3 chunk mainloops + fold + 3 panels + 2 pieces
        assert qg.last_launch_count() == 3 + 1 + 3 + 2


@pytest.mark.parametrize("opA,opB", [("N", "N"), ("T", "H"), ("H", "N")])
def test_host_ragged_k_direct_chunks(opA, opB):
    """K = 1001 (not a multiple of 4): the direct chunk mainloops fall back to the
    32-byte tiles where an operand is k-contiguous; ragged last chunk, M, N not
    multiples of 4 either; exact-integer inputs -> bitwise."""
    pr = make_problem(203, 517, 1001, opA, opB, (2, -1, 0, 3), (1, 0, -2, 1), seed=25, dist="int8")
    assert_parity(pr, run_host(pr), oracle_full(pr), exact=True)


@pytest.mark.parametrize("policy", [qg.PATH_DIRECT, qg.PATH_AUTO], ids=["direct", "auto_packed"])
@pytest.mark.parametrize("opA,opB", [("N", "H"), ("T", "N"), ("H", "T")])
def test_host_f32_chunked(opA, opB, policy):
    """FP32 from host memory: staged K-chunks read in place by the direct pair
    kernel (policy 3) or packed per chunk (auto)."""
    pr = make_problem(260, 700, 900, opA, opB, QALPHA, QBETA, seed=22, dist="normal")
    with path_policy(policy):
        assert_parity(pr, run_host(pr, "f32"), oracle_full(pr), precision="f32")
    pr = make_problem(260, 700, 900, opA, opB, (2, -1, 0, 3), (1, 0, -2, 1), seed=26, dist="int2")
    with path_policy(policy):
        assert_parity(pr, run_host(pr, "f32"), oracle_full(pr), exact=True)


def test_host_beta_zero_nan_c_and_single_chunk():
    """beta = 0: C is never uploaded (NaN host C), K fits one chunk (first == last)."""
    pr = make_problem(400, 300, 200, "N", "H", QALPHA, 0, seed=23, c_init="nan")
    got = run_host(pr)
    assert np.isfinite(got[:, :400]).all()
    assert_parity(pr, got, oracle_full(pr))


def test_host_small_path_and_quick_paths():
    pr = make_problem(64, 64, 64, "N", "N", 1, 0, seed=24)
    assert_parity(pr, run_host(pr), oracle_full(pr))
    assert qg.last_launch_count() == 1  # one-launch small kernel
    with path_policy(qg.PATH_SMALL):
        pr = make_problem(300, 200, 500, "H", "T", QALPHA, QBETA, seed=25, lda=503)
        assert_parity(pr, run_host(pr, pin=False), oracle_full(pr))  # pageable host memory
    # alpha = 0: C <- beta C on the device, no A/B traffic
    pr = make_problem(70, 50, 30, "N", "N", 0, QBETA, seed=26)
    assert_parity(pr, run_host(pr), oracle_full(pr))
    # K = 0
    pr = make_problem(70, 50, 0, "N", "N", 1, QBETA, seed=26)
    assert_parity(pr, run_host(pr), oracle_full(pr))


def test_host_side_stream_and_workspace_errors():
    pr = make_problem(200, 300, 600, "T", "H", QALPHA, QBETA, seed=27)
    need = qg.host_workspace_bytes("T", "H", 200, 300, 600)
    ws = torch.empty(need, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    assert_parity(pr, run_host(pr, stream=s, workspace=ws), oracle_full(pr))
    with pytest.raises(qg.QgemmError) as ei:
        run_host(pr, workspace=ws[: need - 256])
    assert ei.value.code == -15


def test_host_repeated_calls_agree_with_device_path():
    """Back-to-back calls reuse one workspace (stream-ordered), and the host
    path equals the device path bitwise in exact-integer mode (P8)."""
    pr = make_problem(330, 610, 650, "N", "N", (2, -1, 0, 3), (1, 0, -2, 1), seed=28, dist="int8")
    ref = oracle_full(pr)
    for _ in range(3):
        assert_parity(pr, run_host(pr), ref, exact=True)
