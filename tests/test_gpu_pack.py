"""the pack kernel alone (rows a2/a3, Alg. 4 PACK1 /
Alg. 5 PACK2) against a host permutation written from the chunk
layout stated in include/qgemm.h (qgemm_pack_panel) -- bitwise, including the
zero padding of the last row / k tiles, the conj signs of op H
(P:330-334), and NaN in the ld padding (never read)."""
from __future__ import annotations

import ctypes

import numpy as np
import pytest
import torch

import paper_1903_05575_b200 as qg
from synth import quat_matrix

pytestmark = pytest.mark.gpu


def _logical(X: np.ndarray, rows: int) -> np.ndarray:
    """Stored (ncols, ld, 4) -> logical [i, j, c] (rows x ncols)."""
    return X[:, :rows, :].transpose(1, 0, 2)


def host_pack(X: np.ndarray, trans: str, operand: int, R: int, K: int) -> np.ndarray:
    stored_rows = (R if trans == "N" else K) if operand == 0 else (K if trans == "N" else R)
    L = _logical(X, stored_rows)
    if trans != "N":
        L = L.transpose(1, 0, 2).copy()
        if trans == "H":
            L[..., 1:] *= -1.0
    Xt = L if operand == 0 else L.transpose(1, 0, 2)          # X~(r, k): R x K
    assert Xt.shape[:2] == (R, K)
    RT, KT = -(-R // 64), -(-K // 16)
    P = np.zeros((RT * 64, KT * 16, 4))
    P[:R, :K] = Xt
    # r = 64 rt + 8 i + rl, k = 16 kt + 4 ks + kl, c = 2 pp + e, lane = 4 rl + kl
    P = P.reshape(RT, 8, 8, KT, 4, 4, 2, 2)                   # rt i rl kt ks kl pp e
    return P.transpose(0, 3, 4, 1, 6, 2, 5, 7).reshape(-1)    # rt kt ks i pp (rl kl) e


@pytest.mark.parametrize("operand", [0, 1], ids=["A", "B"])
@pytest.mark.parametrize("trans", ["N", "T", "H"])
@pytest.mark.parametrize("R,K", [(64, 16), (130, 37), (7, 100), (200, 5)])
def test_pack_panel_matches_host_permutation(operand, trans, R, K):
    rng = np.random.default_rng(R * 131 + K)
    rows, cols = ((R, K) if trans == "N" else (K, R)) if operand == 0 else \
        ((K, R) if trans == "N" else (R, K))
    X = quat_matrix(rng, rows, cols, rows + 3, "normal")      # NaN in the 3 padding rows
    want = host_pack(X, trans, operand, R, K)
    out = torch.full((want.size,), float("nan"), dtype=torch.float64, device="cuda")
    Xd = torch.from_numpy(X).cuda()
    lib = qg.load()
    rc = lib.qgemm_pack_panel(trans.encode(), operand, R, K, ctypes.c_void_p(Xd.data_ptr()), rows + 3,
                              ctypes.c_void_p(out.data_ptr()), out.numel() * 8,
                              ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert rc == 0
    torch.cuda.synchronize()
    assert lib.qgemm_last_launch_count() == 1
    np.testing.assert_array_equal(out.cpu().numpy(), want)


def test_pack_panel_out_too_small_is_rejected_without_launch():
    X = torch.zeros((16, 64, 4), dtype=torch.float64, device="cuda")
    out = torch.zeros(64 * 16 * 4 - 1, dtype=torch.float64, device="cuda")
    lib = qg.load()
    rc = lib.qgemm_pack_panel(b"N", 0, 64, 16, ctypes.c_void_p(X.data_ptr()), 64,
                              ctypes.c_void_p(out.data_ptr()), out.numel() * 8, None)
    assert rc == -8 and lib.qgemm_last_launch_count() == 0
