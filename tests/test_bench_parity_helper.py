"""CPU checks of bench.py's in-run oracle check (parity_rows_grid), the logic
behind the `parity` / `parity_ok` keys of every bench line: on a small problem
whose 'device result' is the oracle's own full product it passes; one entry off
by more than the tolerance in a checked row, or a row block stored at the wrong
offset, makes it fail."""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import oracle  # noqa: E402


def _setup(world=2, n=96, K=40):
    M = n * world
    A = bench.gen_host(1, np.arange(M), np.arange(K), "normal")        # stored M x K: (K, M, 4)
    B = bench.gen_host(2, np.arange(n), np.arange(K), "normal")        # stored N x K (op H): (K, N, 4)
    C0 = bench.gen_host(3, np.arange(M), np.arange(n), "normal")       # (N, M, 4)
    C = C0.copy()
    oracle.qgemm("N", "H", M, n, K, 1, A, B, 1, C)
    return M, n, K, C

def _check(M, n, K, Cres, world):
    rows = bench.rank_rows(M, world)
    return bench.parity_rows_grid(
        lambda cols, rws: np.ascontiguousarray(Cres[np.asarray(cols)][:, np.asarray(rws)]),
        M, n, K, rows, np.sort(np.random.default_rng(5).choice(M, 16, replace=False)),
        np.sort(np.random.default_rng(6).choice(n, 16, replace=False)),
        lambda r: bench.gen_host(1, r, np.arange(K), "normal"),
        lambda: iter([(0, bench.gen_host(2, np.arange(n), np.arange(K), "normal"))]),
        lambda c: bench.gen_host(2, c, np.arange(K), "normal"),
        lambda r, c: bench.gen_host(3, r, c, "normal"), "H", 1.0, "test")


def test_parity_helper_accepts_the_oracle_product():
    M, n, K, C = _setup()
    res = _check(M, n, K, C, 2)
    assert res["ok"] is True and res["max_err"] <= res["tol"]


def test_parity_helper_rejects_a_wrong_entry_in_a_checked_row():
    M, n, K, C = _setup()
    rows = bench.rank_rows(M, 2)
    bad = C.copy()
    bad[7, rows[-1], 2] += 1e-3                       # column 7 of the last rank's last row
    assert _check(M, n, K, bad, 2)["ok"] is False


def test_parity_helper_rejects_a_misplaced_row_block():
    M, n, K, C = _setup()
    bad = C.copy()
    from paper_1903_05575_b200.dist import rows_for_rank
    r0, _ = rows_for_rank(M, 2, 1)                    # rank 1's block written one row too low
    bad[:, r0 + 1:, :] = C[:, r0:-1, :]
    assert _check(M, n, K, bad, 2)["ok"] is False
    # first, middle and last row of each rank's block of whole 64-row tiles
    assert [int(r) for r in bench.rank_rows(M, 2)] == [0, 65, 127, 128, 161, 191]
