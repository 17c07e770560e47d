"""C-ABI checks that need no GPU (-m "not gpu"): the library builds/loads,
exports every symbol include/qgemm.h declares, and rejects invalid arguments
with LAPACK-style -i codes before touching any device memory."""
from __future__ import annotations

import ctypes
import os
import re
import subprocess

import pytest

from paper_1903_05575_b200 import _lib, build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    build.build()
    return _lib.load()


@pytest.fixture(autouse=True)
def packed_path(lib):
    """The checks below are written for the packed path (workspace arguments);
    the small-problem path is covered by test_small_path_* (policy 2 / auto)."""
    old = lib.qgemm_set_path_policy(1)
    yield
    lib.qgemm_set_path_policy(old)


def _header_symbols():
    txt = open(os.path.join(ROOT, "include", "qgemm.h")).read()
    body = txt[txt.index('extern "C" {'):]
    return set(re.findall(r"\b(q(?:gemm|herk)\w*)\s*\(", body))


def test_exports_match_header(lib):
    declared = _header_symbols()
    assert declared == set(_lib.EXPORTS)
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.SO_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (q(?:gemm|herk)\w*)$", out, re.M))
    assert declared <= exported, declared - exported
    for name in declared:
        assert hasattr(lib, name)


def test_built_for_sm100a(lib):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.SO_PATH],
                         capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out


def test_version(lib):
    assert b"sm_100a" in lib.qgemm_version()


D4 = ctypes.c_double * 4


def _call(lib, tA=b"N", tB=b"N", M=8, N=8, K=8, alpha=1.0, A=0x100000, lda=8, B=0x200000, ldb=8,
          beta=0.0, C=0x300000, ldc=8, ws=0x400000, wsb=1 << 30, stream=None):
    al = D4(alpha, 0, 0, 0) if alpha is not None else None
    be = D4(beta, 0, 0, 0) if beta is not None else None
    return lib.qgemm(tA, tB, M, N, K, ctypes.cast(al, ctypes.c_void_p) if al else None,
                     ctypes.c_void_p(A) if A else None, lda, ctypes.c_void_p(B) if B else None, ldb,
                     ctypes.cast(be, ctypes.c_void_p) if be else None,
                     ctypes.c_void_p(C) if C else None, ldc, ctypes.c_void_p(ws) if ws else None,
                     wsb, stream)


@pytest.mark.parametrize("kw,code", [
    (dict(tA=b"X"), -1), (dict(tB=b"q"), -2), (dict(M=-1), -3), (dict(N=-2), -4),
    (dict(K=-3), -5), (dict(alpha=None), -6), (dict(lda=7), -8), (dict(ldb=7), -10),
    (dict(beta=None), -11), (dict(ldc=7), -13),
    (dict(tA=b"T", M=9, lda=8, ldc=9, ws=None), -14),  # lda >= K ok for T; stops at workspace
    (dict(tA=b"T", K=9, lda=8, ldb=9), -8),                    # T: lda must be >= K
    (dict(tB=b"H", N=9, ldb=8, ldc=8), -10),                   # H: ldb must be >= N
    (dict(A=0x100008), -7), (dict(B=0x200004), -9), (dict(C=0x300008), -12),
    (dict(A=None), -7), (dict(B=None), -9), (dict(C=None), -12),
    (dict(C=0x100000 + 32 * 10), -12),                         # C overlaps A
    (dict(ws=None), -14), (dict(ws=0x400010), -14), (dict(wsb=1000), -15),
])
def test_invalid_arguments(lib, kw, code):
    assert _call(lib, **kw) == code
    assert lib.qgemm_last_launch_count() == 0


def test_lowercase_and_C_alias_accepted_until_workspace(lib):
    # valid shapes with 'c'/'h'/'t' reach the workspace check (-14 with ws=None)
    for t in (b"n", b"t", b"h", b"c", b"C"):
        assert _call(lib, tA=t, tB=t, ws=None) == -14


def test_quick_return_M0_N0(lib):
    assert _call(lib, M=0, A=None, B=None, C=None, ws=None) == 0
    assert _call(lib, N=0, A=None, B=None, C=None, ws=None) == 0
    assert lib.qgemm_last_launch_count() == 0


def test_null_AB_allowed_when_not_read(lib):
    # alpha = 0 or K = 0 never reads A/B: validation passes the A/B checks and
    # would enqueue the beta-scale kernel; check with an invalid C alignment
    # that the first failing argument is C, not A/B.
    assert _call(lib, alpha=0.0, A=None, B=None, C=0x300008) == -12
    assert _call(lib, K=0, A=None, B=None, C=0x300008) == -12


def _herk(lib, uplo=b"L", trans=b"N", N=8, K=8, alpha=1.0, A=0x100000, lda=8, beta=1.0, C=0x300000,
          ldc=8, ws=0x400000, wsb=1 << 30):
    return lib.qherk(uplo, trans, N, K, alpha, ctypes.c_void_p(A) if A else None, lda, beta,
                     ctypes.c_void_p(C) if C else None, ldc, ctypes.c_void_p(ws) if ws else None,
                     wsb, None)


@pytest.mark.parametrize("kw,code", [
    (dict(uplo=b"X"), -1), (dict(trans=b"T"), -2), (dict(N=-1), -3), (dict(K=-1), -4),
    (dict(lda=7), -7), (dict(trans=b"H", K=9, lda=8), -7), (dict(ldc=7), -10),
    (dict(A=0x100008), -6), (dict(A=None), -6), (dict(C=0x300004), -9), (dict(C=None), -9),
    (dict(C=0x100000 + 64), -9), (dict(ws=None), -11), (dict(wsb=100), -12),
    (dict(N=0, A=None, C=None), 0), (dict(alpha=0.0, A=None), 0), (dict(K=0, A=None), 0),
])
def test_qherk_invalid_arguments(lib, kw, code):
    assert _herk(lib, **kw) == code
    assert lib.qgemm_last_launch_count() == 0


# FP32 pair kernel: one raw 4 x 128 x 128 FP32 slot per SM for the accumulation
# chunks (qg_tc32_2cta.cuh), 148 SMs assumed without a device
F32_SLOTS = 148 * 4 * 128 * 128 * 4
# c3 FP32: 2048 tile pairs = 27 waves of 74 + 50; the 50 pairs of the partial
# wave split K 4 ways (200 quarter-K units = 3 waves, cost 0.75 of a whole-pair
# wave), raw partials 50 x 4 x 2 CTAs x (4 x 128 x 128) floats
F32_C3_PART = 50 * 4 * 2 * 4 * 128 * 128 * 4


def test_workspace_sizes(lib):
    old = lib.qgemm_set_path_policy(1)  # the packed path's sizes
    f64 = lib.qgemm_workspace_bytes(b"N", b"H", 8192, 8192, 8192, 0)
    f32 = lib.qgemm_workspace_bytes(b"N", b"H", 8192, 8192, 8192, 1)
    # packed A + B (no padding at tile multiples) + stream-K scratch of the FP64
    # mainloop: 256 partial slots of 128 KiB + 512 arrival counters
    sk = 256 * 131072 + 2048
    assert f64 == 2 * 8192 * 8192 * 32 + sk
    # tcgen05 3xTF32 path: tf32 hi + lo planes + one 256 KiB accumulation-chunk slot
    # per SM (148 assumed without a device)
    assert f32 == 2 * 8192 * 8192 * 32 + F32_SLOTS + F32_C3_PART
    # one K-tile: 2 row tiles of A + 2 of B, 32 KiB per (64 x 16)-quaternion chunk,
    # + partial slots for the largest grid over the whole K (4 tiles x 63 k-tiles
    # / 2 = 126 CTAs) + counters
    assert lib.qgemm_workspace_min_bytes(b"N", b"N", 100, 70, 1000, 0) == 4 * 32768 + 126 * 131072 + 2048
    assert lib.qgemm_workspace_bytes(b"N", b"N", 0, 5, 5, 0) == 0
    assert lib.qgemm_workspace_bytes(b"X", b"N", 5, 5, 5, 0) == 0
    lib.qgemm_set_path_policy(old)


def test_path_policy_setter(lib):
    assert lib.qgemm_set_path_policy(2) == 1
    assert lib.qgemm_set_path_policy(7) == -1  # rejected, unchanged
    assert lib.qgemm_set_path_policy(6) == -1
    assert lib.qgemm_set_path_policy(4) == 2
    assert lib.qgemm_set_path_policy(3) == 4
    assert lib.qgemm_set_path_policy(0) == 3
    assert lib.qgemm_set_path_policy(1) == 0


def test_direct_path_workspace_is_stream_k_scratch(lib):
    """Policy 3 (direct): the pack is fused into the mainloops, so the workspace
    is the FP64 stream-K scratch only (256 partial slots of 128 KiB + 512
    arrival counters), resp. the FP32 pair kernel's accumulation-chunk slots."""
    sk = 256 * 131072 + 2048
    for pol in (3,):
        lib.qgemm_set_path_policy(pol)
        assert lib.qgemm_workspace_bytes(b"N", b"H", 8192, 8192, 8192, 0) == sk
        assert lib.qgemm_workspace_min_bytes(b"N", b"H", 8192, 8192, 8192, 0) == sk
        assert lib.qgemm_workspace_bytes(b"N", b"H", 8192, 8192, 8192, 1) == F32_SLOTS + F32_C3_PART
        assert lib.qherk_workspace_bytes(b"L", b"N", 32768, 256) == sk
    lib.qgemm_set_path_policy(1)  # packed
    assert lib.qherk_workspace_bytes(b"L", b"N", 32768, 256) > sk
    assert lib.qgemm_workspace_bytes(b"N", b"H", 8192, 8192, 8192, 0) > sk
    # auto: direct wherever the 4-quaternion-group tiles apply (c3, c4, c5, QHERK),
    # for op(A) = T/H, and up to 2^37 MACs otherwise; packed for a large ragged op(A) = N
    lib.qgemm_set_path_policy(0)
    assert lib.qherk_workspace_bytes(b"L", b"N", 32768, 256) == sk
    assert lib.qgemm_workspace_bytes(b"N", b"H", 8192, 8192, 8192, 0) == sk
    assert lib.qgemm_workspace_bytes(b"T", b"N", 8192, 8192, 8192, 0) == sk
    assert lib.qgemm_workspace_bytes(b"N", b"N", 1024, 1024, 1024, 0) == sk
    assert lib.qgemm_workspace_bytes(b"N", b"N", 8191, 8192, 8192, 0) > sk   # M % 4 != 0, > 2^37


def test_small_path_needs_no_workspace(lib):
    """Auto policy: below 2^25 quaternion MACs (and for K <= 16 or few-tile long-K
    FP64 shapes) the one-launch kernel is used and no workspace is requested;
    above it the direct / packed path's size is returned."""
    lib.qgemm_set_path_policy(0)
    assert lib.qgemm_workspace_bytes(b"N", b"N", 64, 64, 64, 0) == 0
    assert lib.qgemm_workspace_bytes(b"T", b"H", 320, 320, 320, 1) == 0   # FP32: <= 2^25
    assert lib.qgemm_workspace_bytes(b"T", b"H", 384, 384, 384, 1) > 0    # FP32 above: packed (split K)
    assert lib.qgemm_workspace_bytes(b"N", b"N", 64, 64, 4096, 1) == 0    # FP32: one pair, long K
    assert lib.qgemm_workspace_bytes(b"N", b"N", 320, 320, 320, 0) == 0   # FP64: <= 2^25
    assert lib.qgemm_workspace_bytes(b"N", b"N", 384, 384, 384, 0) > 0    # FP64 above: direct
    assert lib.qgemm_workspace_bytes(b"N", b"N", 64, 64, 8192, 0) == 0    # few tiles, long K
    assert lib.qgemm_workspace_bytes(b"N", b"N", 4096, 4096, 2, 0) == 0   # K <= 16
    assert lib.qgemm_workspace_bytes(b"N", b"H", 8192, 8192, 8192, 0) > 0
    # huge single factors must not overflow M*N*K into the small path
    assert lib.qgemm_workspace_bytes(b"N", b"N", 1 << 40, 1 << 40, 1, 0) > 0
    lib.qgemm_set_path_policy(2)
    assert lib.qgemm_workspace_bytes(b"N", b"H", 8192, 8192, 8192, 0) == 0


@pytest.mark.parametrize("kw,code", [
    (dict(tA=b"X"), -1), (dict(tB=b"q"), -2), (dict(M=-1), -3), (dict(N=-2), -4),
    (dict(K=-3), -5), (dict(alpha=None), -6), (dict(lda=7), -8), (dict(ldb=7), -10),
    (dict(beta=None), -11), (dict(ldc=7), -13), (dict(tA=b"T", K=9, lda=8, ldb=9), -8),
    (dict(A=0x100008), -7), (dict(B=0x200004), -9), (dict(C=0x300008), -12),
    (dict(A=None), -7), (dict(B=None), -9), (dict(C=None), -12),
    (dict(C=0x100000 + 32 * 10), -12),
])
def test_small_path_validates_identically(lib, kw, code):
    lib.qgemm_set_path_policy(2)
    assert _call(lib, ws=None, wsb=0, **kw) == code
    assert lib.qgemm_last_launch_count() == 0


def test_host_workspace_c3_plan(lib):
    """qgemm_host at c3 (FP64, auto = direct chunks): caller's C + accumulator C
    (2 x 2 GiB) + 2 staging slots per operand for the largest K-chunk (4096 k:
    chunks 256, 1024, 2048, 768, 4096 after the longest-last reorder) + the
    stream-K scratch; no packed buffers (the chunks are read in place)."""
    lib.qgemm_set_path_policy(0)
    n = 8192
    sk = 256 * 131072 + 2048
    assert lib.qgemm_host_workspace_bytes(b"N", b"H", n, n, n, 0) == 2 * n * n * 32 + 4 * n * 4096 * 32 + sk
    old = lib.qgemm_set_path_policy(1)  # packed chunks: + 2 packed chunks per operand
    assert lib.qgemm_host_workspace_bytes(b"N", b"H", n, n, n, 0) == 2 * n * n * 32 + 8 * n * 4096 * 32 + sk
    lib.qgemm_set_path_policy(old)


@pytest.mark.parametrize("N", [8192, 1024])
@pytest.mark.parametrize("policy", [1, 3], ids=["packed", "direct"])
def test_host_workspace_f32_covers_every_panel_split(lib, N, policy):
    """qgemm_host_f32 (M = K = 8192): the last chunk runs per column panel and
    its last panel in 128-column pieces; a 128-wide piece has 32 tile pairs
    (< one wave of 74) and splits K twice, so the plan must reserve its split-K
    partials (32 pairs x 2 splits x 512 KiB = 32 MiB) even though the full width
    and the panel width do not split.  (The reserve used to cover only the full
    and the panel width: an out-of-bounds write of 32 MiB.)  Packed chunks
    (policy 1, and auto for FP32) also hold 2 packed chunks per operand; the
    direct chunks (policy 3) are read in place from the staging slots.
    Above one wave only the pairs of the partial last wave split:
    N = 8192's 512-wide panels have 128 pairs = 74 + 54, split 4 ways (54 x 4
    units = 3 waves); N = 1024's full width has 256 pairs = 3 x 74 + 34, split 2
    ways.  Those exceed the 128-wide pieces' 32 x 2 units."""
    lib.qgemm_set_path_policy(policy)
    M = K = 8192
    qb = 16
    kc = 4096                                    # chunks 256, 1024, 2048, 768, 4096
    stage = 2 * M * kc * qb + 2 * N * kc * qb
    ktc = kc // 8                                # FP32 k-tiles per chunk (8 k per tile)
    packed = 2 * (2 * (M // 256)) * ktc * 32768 + 2 * (N // 128) * ktc * 32768
    units = {8192: 54 * 4, 1024: 34 * 2}[N]      # split pairs x S, the largest of any launched width
    part = units * 2 * 65536 * 4                 # x 2 CTAs x 4x128x128 floats
    want = 2 * M * N * qb + stage + (packed if policy == 1 else 0) + F32_SLOTS + part
    assert lib.qgemm_host_workspace_bytes(b"N", b"H", M, N, K, 1) == want
    lib.qgemm_set_path_policy(1)


@pytest.mark.parametrize("args,code", [
    ((b"X", 0, 64, 16, 0x1000, 64, 0x2000, 1 << 20), -1),
    ((b"N", 2, 64, 16, 0x1000, 64, 0x2000, 1 << 20), -2),
    ((b"N", 0, -1, 16, 0x1000, 64, 0x2000, 1 << 20), -3),
    ((b"N", 0, 64, -1, 0x1000, 64, 0x2000, 1 << 20), -4),
    ((b"N", 0, 64, 16, 0x1008, 64, 0x2000, 1 << 20), -5),
    ((b"N", 0, 64, 16, 0x1000, 63, 0x2000, 1 << 20), -6),
    ((b"T", 0, 64, 16, 0x1000, 15, 0x2000, 1 << 20), -6),
    ((b"N", 1, 64, 16, 0x1000, 15, 0x2000, 1 << 20), -6),
    ((b"N", 0, 64, 16, 0x1000, 64, None, 1 << 20), -7),
    ((b"N", 0, 64, 16, 0x1000, 64, 0x2000, 64 * 16 * 32 - 1), -8),
    ((b"N", 0, 0, 16, None, 64, None, 0), 0),
])
def test_pack_panel_validation(lib, args, code):
    """qgemm_pack_panel (the a2/a3 test hook): every error code, nothing enqueued."""
    tr, operand, R, K, X, ldx, out, nbytes = args
    assert lib.qgemm_pack_panel(tr, operand, R, K, X, ldx, out, nbytes, None) == code
    assert lib.qgemm_last_launch_count() == 0
