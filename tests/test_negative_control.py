"""Negative control: a library built with ONE flipped sign in
the Hamilton product table (eps(1,2), -DQG_NEGATIVE_CONTROL) must fail the
parity check the real library passes -- evidence that the parity tests can see
a single wrong term.  The variant is built into a temp dir and driven through
the same C ABI with ctypes; libqgemm.so itself is never built this way."""
from __future__ import annotations

import ctypes

import numpy as np
import pytest

import oracle
from paper_1903_05575_b200 import build
from synth import make_problem


@pytest.fixture(scope="module")
def bad_lib(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("negctl") / "libqgemm_negative_control.so")
    build.build_variant(out, ["-DQG_NEGATIVE_CONTROL"])
    return out


def test_negative_control_builds(bad_lib):
    lib = ctypes.CDLL(bad_lib)
    assert lib.qgemm_version  # same ABI


@pytest.mark.gpu
@pytest.mark.parametrize("policy", [1, 2, 3])  # packed, small kernel, direct
def test_flipped_sign_fails_parity(bad_lib, policy):
    import torch
    lib = ctypes.CDLL(bad_lib)
    vp = ctypes.c_void_p
    lib.qgemm.argtypes = [ctypes.c_char, ctypes.c_char] + [ctypes.c_int64] * 3 + [
        vp, vp, ctypes.c_int64, vp, ctypes.c_int64, vp, vp, ctypes.c_int64, vp, ctypes.c_size_t, vp]
    lib.qgemm_workspace_bytes.restype = ctypes.c_size_t
    lib.qgemm_workspace_bytes.argtypes = [ctypes.c_char, ctypes.c_char] + [ctypes.c_int64] * 3 + [ctypes.c_int]
    lib.qgemm_set_path_policy(policy)
    M, N, K = 300, 200, 256
    pr = make_problem(M, N, K, "N", "N", (1, 0, 0, 0), (0, 0, 0, 0), seed=1, dist="int8")
    A, B = (torch.from_numpy(x).cuda() for x in (pr.A, pr.B))
    C = torch.zeros_like(torch.from_numpy(pr.C)).cuda()
    ws = torch.empty(max(256, lib.qgemm_workspace_bytes(b"N", b"N", M, N, K, 0)), dtype=torch.uint8,
                     device="cuda")
    one = (ctypes.c_double * 4)(1, 0, 0, 0)
    zero = (ctypes.c_double * 4)(0, 0, 0, 0)
    rc = lib.qgemm(b"N", b"N", M, N, K, ctypes.cast(one, vp), vp(A.data_ptr()), M, vp(B.data_ptr()), K,
                   ctypes.cast(zero, vp), vp(C.data_ptr()), M, vp(ws.data_ptr()), ws.numel(),
                   vp(torch.cuda.current_stream().cuda_stream))
    assert rc == 0
    torch.cuda.synchronize()
    ref = pr.C.copy()
    oracle.qgemm("N", "N", M, N, K, pr.alpha, pr.A, pr.B, pr.beta, ref)
    got = C.cpu().numpy()
    # exact-integer data: the real library is bitwise equal (test_gpu_parity);
    # the flipped sign must show up as a large error in components 3 (= 1 xor 2)
    err = np.abs(got[:, :M] - ref[:, :M])
    assert err[..., 3].max() > 1.0 and err[..., :3].max() == 0.0
