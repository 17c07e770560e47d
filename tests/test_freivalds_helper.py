"""CPU checks of the block Freivalds helper (tests/freivalds.py) on the oracle's
own results: the residual of a correct C is at rounding level, and one entry
moved by d moves exactly the residual of its (row, column block) by d x_j."""
from __future__ import annotations

import numpy as np

import oracle
from synth import make_problem
from tests.freivalds import Check, blocks, columns_of, draw_x, qnorm, times_x


def _setup(opB, bs):
    pr = make_problem(40, 50, 30, "N", opB, (0.5, 1, 0, -2), (1, 0, 0.5, 0), seed=2, dist="normal")
    C = pr.C.copy()
    oracle.qgemm("N", opB, pr.M, pr.N, pr.K, pr.alpha, pr.A, pr.B, pr.beta, C)
    x = draw_x(pr.N, seed=3)
    if opB == "N":
        getb = lambda j0, j1: (pr.B[j0:j1], "N")          # noqa: E731
    else:
        getb = lambda j0, j1: (pr.B[:, j0:j1, :], opB)    # noqa: E731
    Y = times_x(getb, pr.K, pr.N, x, bs)
    AY = np.zeros((Y.shape[0], pr.M, 4))
    oracle.qgemm("N", "N", pr.M, Y.shape[0], pr.K, pr.alpha, pr.A, Y, 0, AY)
    C0X = times_x(columns_of(pr.C), pr.M, pr.N, x, bs)
    BC0X = np.stack([np.array([oracle.hmul(pr.beta, q) for q in v]) for v in C0X])  # beta from the left
    return pr, C, x, Check(pr.M, pr.N, bs, x, AY + BC0X)


def test_block_freivalds_correct_c_is_rounding_level():
    for opB in ("N", "H", "T"):
        pr, C, x, chk = _setup(opB, bs=7)
        assert len(blocks(pr.N, 7)) == 8
        assert qnorm(chk.residual(columns_of(C))).max() < 1e-12


def test_block_freivalds_locates_a_wrong_entry():
    pr, C, x, chk = _setup("H", bs=7)
    bad = C.copy()
    d = np.array([0.0, 1e-3, 0.0, 0.0])
    bad[23, 11] += d                                      # column 23, row 11
    R = chk.residual(columns_of(bad))
    v = 23 // 7
    assert abs(qnorm(R[v, 11]) - 1e-3 * qnorm(x[23])) < 1e-12
    mask = np.ones(R.shape[:2], dtype=bool)
    mask[v, 11] = False
    assert qnorm(R[mask]).max() < 1e-12
    # calibrated bound from rows known exactly: the wrong entry exceeds it
    rows = np.array([0, 5, 39])
    b = chk.bound(np.ascontiguousarray(C[:, rows, :]), np.ascontiguousarray(C[:, rows, :]), rows)
    assert b < 1e-3 < qnorm(R).max()
