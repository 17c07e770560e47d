"""Parity at BASELINE.json's full sizes for configs 4 and 5 (-m gpu).

Inputs come from the counter-based generator (synth/gpu_gen.py) so the host can
regenerate exactly the rows/columns the oracle needs; outputs are compared on
sampled entries computed by the oracle one by one, plus properties that hold at
any size (Hermiticity for c4; finiteness with a NaN-filled C and
beta = 0 for c5); c4 is also checked in full, every entry against the oracle
(~2.5 minutes).  c5 runs with a 16 GB workspace, i.e. through the K-panel loop.
"""
from __future__ import annotations

import numpy as np
import pytest
import torch

import oracle
import paper_1903_05575_b200 as qg
from synth.gpu_gen import (counter_hermitian, counter_matrix, counter_uniform_t, host_cols,
                           host_hermitian_entries, host_rows_N)
from synth.inputs import counter_uniform

pytestmark = pytest.mark.gpu


def test_counter_generator_device_matches_host():
    idx = np.random.default_rng(0).integers(0, 1 << 40, 100000)
    dev = counter_uniform_t(7, 3, torch.from_numpy(idx).cuda()).cpu().numpy()
    np.testing.assert_array_equal(dev, counter_uniform(7, 3, idx))


def _free():
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


def test_c4_full_size_hermitian_rank_k():
    """c4: M = N = 32768, K = 256, C <- A A^H + C, B == A (same buffer), C Hermitian."""
    n, K = 32768, 256
    A = counter_matrix(0, 1, n, K, "cuda")            # stored n x K (op N), ld = n
    C = counter_hermitian(0, 3, n, "cuda")
    qg.qgemm("N", "H", 1.0, A, A, 1.0, C, M=n, N=n, K=K)
    torch.cuda.synchronize()
    maxa = float(A.abs().max())
    maxc0 = 1.0
    tol = 1e-12 * K * maxa * maxa + 8 * 2.0 ** -53 * maxc0 * 4
    # P12: the result is Hermitian, checked over the full matrix on the device
    sign = torch.tensor([1.0, -1.0, -1.0, -1.0], dtype=torch.float64, device="cuda")
    herm = 0.0
    for j0 in range(0, n, 1024):
        blk = C[j0:j0 + 1024]                                # columns j0.., all rows: C_ij
        tr = C[:, j0:j0 + 1024, :].transpose(0, 1)           # C_ji for the same (i, j)
        herm = max(herm, float((blk - sign * tr).abs().max()))
    assert herm <= 2 * tol, (herm, tol)
    # sampled entries vs the oracle: 2 full rows, 2 full columns, 256 random
    A_h = counter_matrix(0, 1, n, K, "cpu").numpy()
    rng = np.random.default_rng(4)
    rows = np.concatenate([np.full(n, 3), np.full(n, n - 1), np.arange(n), np.arange(n),
                           rng.integers(0, n, 256)])
    cols = np.concatenate([np.arange(n), np.arange(n), np.full(n, 0), np.full(n, n - 7),
                           rng.integers(0, n, 256)])
    t = oracle.qgemm_entries("N", "H", n, n, K, 1, A_h, A_h, 0, None, rows, cols)
    ref = t + host_hermitian_entries(0, 3, n, rows, cols)    # alpha = 1, beta = 1 (real)
    got = C[torch.from_numpy(cols).cuda(), torch.from_numpy(rows).cuda()].cpu().numpy()
    err = float(np.abs(got - ref).max())
    assert err <= tol, (err, tol)
    del A, C
    _free()


def test_c4_full_size_every_entry_vs_oracle():
    """c4 in full (SURVEY §8(c) coverage table: 'c4 full (8.8e12 flops) + P12'):
    every one of the 32768^2 entries against the oracle, 1024 columns at a time
    (the oracle runs on all host cores; ~2.5 minutes on a 16-core host).  C0 is the
    counter-generated Hermitian matrix (the seeded generator's torch twin, bitwise
    equal to the host one: test_counter_generator_device_matches_host), copied to
    the host block by block."""
    n, K, blk = 32768, 256, 1024
    A = counter_matrix(0, 1, n, K, "cuda")
    C0 = counter_hermitian(0, 3, n, "cuda")
    C = C0.clone()
    qg.qgemm("N", "H", 1.0, A, A, 1.0, C, M=n, N=n, K=K)
    torch.cuda.synchronize()
    A_h = counter_matrix(0, 1, n, K, "cpu").numpy()        # stored n x K: (K, n, 4), host generator
    maxa = float(np.abs(A_h).max())
    tol = 1e-12 * K * maxa * maxa + 8 * 2.0 ** -53 * float(C0.abs().max()) * 4
    worst = 0.0
    for j0 in range(0, n, blk):
        # columns j0.. of op(B) = A^H are rows j0.. of stored A, op H
        B_blk = np.ascontiguousarray(A_h[:, j0:j0 + blk, :])   # (K, blk, 4)
        ref = C0[j0:j0 + blk].cpu().numpy()                    # (blk, n, 4), beta = 1
        oracle.qgemm("N", "H", n, blk, K, 1, A_h, B_blk, 1, ref)
        got = C[j0:j0 + blk].cpu().numpy()
        worst = max(worst, float(np.abs(got - ref).max()))
        assert worst <= tol, (j0, worst, tol)
    del A, C0, C
    _free()


@pytest.mark.parametrize("mode", ["packed_kpanels", "auto_direct"])
def test_c5_full_size_kpanel_nan_c(mode):
    """c5: M = N = K = 32768, N/N, alpha = 1, beta = 0 with C NaN-filled; either the
    packed path with a 16 GB workspace (K-panel loop) or the auto path (TMA-fed
    mainloop, one launch, stream-K scratch only); 66 x 66 sampled entries (incl.
    first/last row/column) from the oracle on host-regenerated rows of A / columns of B."""
    n = 32768
    A = counter_matrix(0, 1, n, n, "cuda")
    B = counter_matrix(0, 2, n, n, "cuda")
    C = torch.full((n, n, 4), float("nan"), dtype=torch.float64, device="cuda")
    if mode == "packed_kpanels":
        ws_bytes = 16 * 10 ** 9
        old = qg.set_path_policy(qg.PATH_PACKED)
        try:
            assert ws_bytes < qg.workspace_bytes("N", "N", n, n, n)
            ws = torch.empty(ws_bytes, dtype=torch.uint8, device="cuda")
            qg.qgemm("N", "N", 1.0, A, B, 0.0, C, workspace=ws)
            torch.cuda.synchronize()
            assert qg.last_launch_count() > 3      # several K-panels
        finally:
            qg.set_path_policy(old)
    else:
        ws = None
        qg.qgemm("N", "N", 1.0, A, B, 0.0, C)
        torch.cuda.synchronize()
        assert qg.last_launch_count() == 1         # no pack, no K-panels
    assert bool(torch.isfinite(C).all())          # beta = 0: C never read (R3)
    rng = np.random.default_rng(5)
    rows = np.concatenate([[0, n - 1], rng.integers(0, n, 64)])
    cols = np.concatenate([[0, n - 1], rng.integers(0, n, 64)])
    A_rows = host_rows_N(0, 1, n, rows, n)     # op(A) rows: stored (K, |R|, 4)
    B_cols = host_cols(0, 2, n, cols, n)       # op(B) columns: stored (|S|, K, 4)
    ref = np.zeros((cols.size, rows.size, 4))
    oracle.qgemm("N", "N", rows.size, cols.size, n, 1, np.ascontiguousarray(A_rows), B_cols, 0, ref)
    got = C[torch.from_numpy(cols).cuda()][:, torch.from_numpy(rows).cuda()].cpu().numpy()
    tol = 1e-12 * n * max(np.abs(A_rows).max(), 1e-300) * np.abs(B_cols).max()
    # max over the sampled operands is <= the global max: a stricter tolerance
    err = float(np.abs(got - ref).max())
    assert err <= tol, (err, tol)
    del A, B, C, ws
    _free()
