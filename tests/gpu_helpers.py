"""Helpers for the -m gpu parity tests: move synth problems to the device, run
the C-ABI path, compare with the oracle (tests only)."""
from __future__ import annotations

import contextlib

import numpy as np
import torch

import oracle
import paper_1903_05575_b200 as qg
from tests.tolerance import tolerance


@contextlib.contextmanager
def path_policy(policy):
    """Force the packed (1) or the one-launch small (2) path for the block."""
    old = qg.set_path_policy(policy)
    try:
        yield
    finally:
        qg.set_path_policy(old)


def to_dev(x: np.ndarray, dtype=torch.float64) -> torch.Tensor:
    return torch.from_numpy(np.ascontiguousarray(x)).to(device="cuda", dtype=dtype)


def run_gpu(pr, precision="f64", workspace=None, naive=False, stream=None):
    """Run the problem through the library; returns the full stored C (numpy f64)."""
    dt = torch.float64 if precision == "f64" else torch.float32
    A = to_dev(pr.A, dt)
    B = A if pr.B is pr.A else to_dev(pr.B, dt)
    C = to_dev(pr.C, dt)
    if naive:
        qg.qgemm_naive(pr.transA, pr.transB, pr.alpha, A, B, pr.beta, C, M=pr.M, N=pr.N, K=pr.K,
                       stream=stream)
    else:
        fn = qg.qgemm if precision == "f64" else qg.qgemm_f32
        fn(pr.transA, pr.transB, pr.alpha, A, B, pr.beta, C, M=pr.M, N=pr.N, K=pr.K,
           workspace=workspace, stream=stream)
    torch.cuda.synchronize()
    return C.double().cpu().numpy()


def oracle_full(pr):
    C = pr.C.copy()
    oracle.qgemm(pr.transA, pr.transB, pr.M, pr.N, pr.K, pr.alpha, pr.A, pr.B, pr.beta, C)
    return C


def tol_for(pr, precision):
    a_rows = pr.M if pr.transA == "N" else pr.K
    b_rows = pr.K if pr.transB == "N" else pr.N
    return tolerance(precision, pr.K, pr.A, a_rows, pr.B, b_rows, pr.beta, pr.C, pr.M)


def assert_parity(pr, got, ref, precision="f64", exact=False):
    """Element-by-element on the logical M x N block; ld padding must be untouched."""
    g = got[:, : pr.M, :]
    r = ref[:, : pr.M, :]
    if exact:
        np.testing.assert_array_equal(g, r)
    else:
        tol = tol_for(pr, precision)
        err = float(np.max(np.abs(g - r))) if g.size else 0.0
        assert np.all(np.isfinite(g)), "non-finite output"
        assert err <= tol, f"max|C - C_ref| = {err:.3e} > tol {tol:.3e}"
    # padding rows of C never written (sentinel preserved, NaN-safe compare)
    np.testing.assert_array_equal(got[:, pr.M:, :], pr.C[:, pr.M:, :])
