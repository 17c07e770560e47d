"""Host logic of the row-block multi-GPU driver (dist.py) on CPU with gloo,
world_size 2 (-m "not gpu").  The local GEMM is injected (the oracle on CPU
tensors) -- this exercises sharding, the broadcast of B, the gather and the
strided relayout of C only; the GPU product path is tested in -m gpu."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1903_05575_b200.dist import qgemm_rowsharded, rows_for_rank
from synth import make_problem


def test_rows_for_rank_partition():
    for M in (1, 63, 64, 65, 1000, 8192 * 3 + 5):
        for world in (1, 2, 3, 4, 8):
            blocks = [rows_for_rank(M, world, r) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == M
            for (a0, a1), (b0, b1) in zip(blocks, blocks[1:]):
                assert a1 == b0 and a0 <= a1
            sizes = [b - a for a, b in blocks]
            # whole 64-row tiles except the global tail; balanced within one tile
            assert all(a % 64 == 0 or a == M for a, _ in blocks)
            assert max(sizes) - min(sizes) <= 64 + 63


def _oracle_local(transA, transB, alpha, A, B, beta, C, M, N, K):
    a, b, c = A.numpy(), B.numpy(), C.numpy()
    oracle.qgemm(transA, transB, M, N, K, alpha, np.ascontiguousarray(a), np.ascontiguousarray(b),
                 beta, c)  # C is contiguous -> updated in place through the numpy view


def _worker(rank, world, port, opA, opB, M, N, K, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        pr = make_problem(M, N, K, opA, opB, (0.5, 0.25, -1, 0.1), (1, -0.5, 0, 0.2), seed=3)
        r0, r1 = rows_for_rank(M, world, rank)
        # this rank's stored operand: op(A_local) = rows [r0, r1) of op(A)
        if opA == "N":
            A_loc = np.ascontiguousarray(pr.A[:, r0:r1, :])          # (K, m_loc, 4)
        else:
            A_loc = np.ascontiguousarray(pr.A[r0:r1, :, :])          # (m_loc, K, 4)
        C_loc = pr.C[:, r0:r1, :].copy()  # never a view of pr.C (used for the reference)
        B = torch.from_numpy(pr.B.copy()) if rank == 0 else torch.full(pr.B.shape, np.nan,
                                                                        dtype=torch.float64)
        C_full = torch.full((N, M, 4), np.nan, dtype=torch.float64) if rank == 0 else None
        out = qgemm_rowsharded(opA, opB, pr.alpha, torch.from_numpy(A_loc), B, pr.beta,
                               torch.from_numpy(C_loc), M, N, K, C_full=C_full,
                               local_gemm=_oracle_local)
        if rank == 0:
            ref = pr.C.copy()
            oracle.qgemm(opA, opB, M, N, K, pr.alpha, pr.A, pr.B, pr.beta, ref)
            # same per-entry summation order -> bitwise equal to the unsharded oracle
            q.put(bool(np.array_equal(out.numpy(), ref)))
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("opA,opB,M", [("N", "H", 150), ("H", "N", 130), ("T", "T", 64)])
def test_rowsharded_gloo_world2(opA, opB, M):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    N, K = 37, 29
    procs = [ctx.Process(target=_worker, args=(r, 2, port, opA, opB, M, N, K, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert q.get(timeout=5) is True


# ---------------------------------------------------------------- fused collection (p2p)
def _raw(addr, ncols, ld, nrows=None):
    """(ncols, nrows, 4) float64 numpy view of the column-major matrix at `addr`
    with leading dimension ld (only the addressed elements: no read past the
    last column's rows)."""
    import ctypes
    nrows = ld if nrows is None else nrows
    flat = np.ctypeslib.as_array(ctypes.cast(addr, ctypes.POINTER(ctypes.c_double)),
                                 shape=(4 * ((ncols - 1) * ld + nrows),))
    return np.lib.stride_tricks.as_strided(flat, shape=(ncols, nrows, 4), strides=(32 * ld, 32, 8))


def _oracle_local_ptr(transA, transB, m_loc, N, K, alpha, A, lda, B, ldb, beta, c_addr, ldc):
    """Local GEMM on raw addresses with the leading dimensions the driver passes
    (exactly what reaches the C ABI): A and B read through (data_ptr, ld), root's
    C written at rows r0.. of a column-major matrix with leading dimension ldc --
    the CPU stand-in for the epilogue storing over peer memory.  Only the first
    (cols - 1) * ld + rows quaternions of each operand are addressed."""
    a_cols = K if transA == "N" else m_loc
    a_rows = m_loc if transA == "N" else K
    b_cols = N if transB == "N" else K
    b_rows = K if transB == "N" else N
    Av = np.ascontiguousarray(_raw(A.data_ptr(), a_cols, lda, a_rows))
    Bv = np.ascontiguousarray(_raw(B.data_ptr(), b_cols, ldb, b_rows))
    # root's C from this rank's row r0 on, ld = ldc (the oracle reads ldc from
    # the shape; it touches rows [0, m_loc) of each column only)
    import ctypes
    Cv = np.ctypeslib.as_array(ctypes.cast(c_addr, ctypes.POINTER(ctypes.c_double)), shape=(N, ldc, 4))
    oracle.qgemm(transA, transB, m_loc, N, K, alpha, Av, Bv, beta, Cv)


def _p2p_worker(rank, world, port, opA, opB, M, N, K, path, q, view=False):
    from paper_1903_05575_b200.dist import PeerC, qgemm_rowsharded_p2p
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        pr = make_problem(M, N, K, opA, opB, (0.5, 0.25, -1, 0.1), (1, -0.5, 0, 0.2), seed=5,
                          ldc=M + 3)
        r0, r1 = rows_for_rank(M, world, rank)
        A_full = torch.from_numpy(pr.A.copy())
        if view:  # a strided row-block view of the stored A: lda = M, from the strides
            A_loc = A_full[:, r0:r1, :] if opA == "N" else A_full[r0:r1]
            assert opA != "N" or not A_loc.is_contiguous()
        else:
            A_loc = (torch.from_numpy(np.ascontiguousarray(pr.A[:, r0:r1, :])) if opA == "N"
                     else torch.from_numpy(np.ascontiguousarray(pr.A[r0:r1, :, :])))
        B = torch.from_numpy(pr.B.copy()) if rank == 0 else torch.full(pr.B.shape, np.nan,
                                                                        dtype=torch.float64)
        n_el = pr.C.size
        keep = []

        def share(t):
            return path

        def open_(p):
            t = torch.from_file(p, shared=True, size=n_el, dtype=torch.float64)
            keep.append(t)
            return t.data_ptr(), t

        C_root = None
        if rank == 0:  # root's C (ld = M + 3, padding sentinel) in a shared file
            C_root = torch.from_file(path, shared=True, size=n_el, dtype=torch.float64)
            C_root.copy_(torch.from_numpy(pr.C.reshape(-1)))
            C_root = C_root.view(pr.C.shape)
        peer = PeerC(C_root, share=share, open_=open_, close=lambda b: None)
        assert peer.ldc == M + 3 and peer.ncols == N
        qgemm_rowsharded_p2p(opA, opB, pr.alpha, A_loc, B, pr.beta, peer, M, N,
                             K, local_gemm_ptr=_oracle_local_ptr)
        if rank == 0:
            ref = pr.C.copy()
            oracle.qgemm(opA, opB, M, N, K, pr.alpha, pr.A, pr.B, pr.beta, ref)
            q.put(bool(np.array_equal(C_root.numpy(), ref)))  # incl. untouched ld padding
        peer.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("opA,opB,M,view", [("N", "H", 150, False), ("H", "T", 130, False),
                                             ("N", "H", 150, True), ("T", "N", 130, True)])
def test_rowsharded_p2p_gloo_world2(opA, opB, M, view, tmp_path):
    """view=True: each rank hands the driver a strided row-block VIEW of the full
    stored A (SURVEY §8(e)'s c4 layout, lda = M); the leading dimension must come
    from the strides (a shape-derived lda = m_loc reads the wrong elements)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    N, K = 37, 29
    path = str(tmp_path / "c_root.bin")
    procs = [ctx.Process(target=_p2p_worker, args=(r, 2, port, opA, opB, M, N, K, path, q, view))
             for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert q.get(timeout=5) is True


# ---------------------------------------------------------------- c4 structure: B == A, A_r a view
def _c4_worker(rank, world, port, M, K, path, q):
    """C <- A A^H + C with B == A (the broadcast operand) and each rank's A_r a
    strided view of it (rows [r0, r1), lda = M): SURVEY §8(e)'s c4 layout."""
    from paper_1903_05575_b200.dist import PeerC, qgemm_rowsharded_p2p
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        pr = make_problem(M, M, K, "N", "H", 1, 1, seed=8, c_init="hermitian", b_is_a=True)
        r0, r1 = rows_for_rank(M, world, rank)
        A = torch.from_numpy(pr.A.copy()) if rank == 0 else torch.full(pr.A.shape, np.nan,
                                                                        dtype=torch.float64)
        n_el = pr.C.size
        keep = []

        def open_(p):
            t = torch.from_file(p, shared=True, size=n_el, dtype=torch.float64)
            keep.append(t)
            return t.data_ptr(), t

        C_root = None
        if rank == 0:
            C_root = torch.from_file(path, shared=True, size=n_el, dtype=torch.float64)
            C_root.copy_(torch.from_numpy(pr.C.reshape(-1)))
            C_root = C_root.view(pr.C.shape)
        peer = PeerC(C_root, share=lambda t: path, open_=open_, close=lambda b: None)
        # the broadcast of B (== A) fills A on every rank before the view is read
        qgemm_rowsharded_p2p("N", "H", 1, A[:, r0:r1, :], A, 1, peer, M, M, K,
                             local_gemm_ptr=_oracle_local_ptr)
        if rank == 0:
            ref = pr.C.copy()
            oracle.qgemm("N", "H", M, M, K, 1, pr.A, pr.A, 1, ref)
            q.put(bool(np.array_equal(C_root.numpy(), ref)))
        peer.close()
    finally:
        dist.destroy_process_group()


def test_rowsharded_p2p_c4_structure_gloo_world2(tmp_path):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    path = str(tmp_path / "c_root.bin")
    procs = [ctx.Process(target=_c4_worker, args=(r, 2, port, 192, 24, path, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert q.get(timeout=5) is True
