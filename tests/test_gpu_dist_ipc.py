"""Fused collection of the row-sharded QGEMM over peer memory (-m gpu).

Two processes share cuda:0 (the GPU box has one GPU): rank 1 maps rank 0's C
with the library's CUDA IPC calls (qgemm_ipc_handle / qgemm_ipc_open) and its
QGEMM epilogue stores its row block straight into rank 0's allocation; rank 0
computes its own block in place.  The two ranks' kernels never wait on each
other (the host-side gloo all_reduce after the local QGEMM is the only
synchronisation), so this is a functional test of the IPC mapping, the row
offset and root's leading dimension -- not a stand-in for NVLink timing.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from synth import make_problem
from tests.tolerance import tolerance

pytestmark = pytest.mark.gpu


def _worker(rank, world, port, opA, opB, M, N, K, q, dist_kind="normal"):
    import paper_1903_05575_b200 as qg
    from paper_1903_05575_b200.dist import PeerC, qgemm_rowsharded_p2p, rows_for_rank
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        exact = dist_kind == "int8"
        pr = make_problem(M, N, K, opA, opB, (2, -1, 0, 1) if exact else (0.5, 0.25, -1, 0.1),
                          (1, 0, -1, 0) if exact else (1, -0.5, 0, 0.2), seed=7, dist=dist_kind, ldc=M + 5)
        r0, r1 = rows_for_rank(M, world, rank)
        A_loc = (np.ascontiguousarray(pr.A[:, r0:r1, :]) if opA == "N"
                 else np.ascontiguousarray(pr.A[r0:r1, :, :]))
        dev = torch.device("cuda", 0)
        A_d = torch.from_numpy(A_loc).to(dev)
        B_d = (torch.from_numpy(pr.B.copy()).to(dev) if rank == 0
               else torch.full(pr.B.shape, float("nan"), dtype=torch.float64, device=dev))
        # root's C lives inside a larger allocation: the handle's offset is exercised
        C_big = None
        C_root = None
        if rank == 0:
            C_big = torch.full((pr.C.size + 1000,), float("nan"), dtype=torch.float64, device=dev)
            C_root = C_big[1000:].view(pr.C.shape)
            C_root.copy_(torch.from_numpy(pr.C))
        peer = PeerC(C_root)
        for _ in range(2):  # repeated steps reuse the mapping (C accumulates)
            qgemm_rowsharded_p2p(opA, opB, pr.alpha, A_d, B_d, pr.beta, peer, M, N, K)
        torch.cuda.synchronize()
        dist.barrier()
        if rank == 0:
            ref = pr.C.copy()
            for _ in range(2):
                oracle.qgemm(opA, opB, M, N, K, pr.alpha, pr.A, pr.B, pr.beta, ref)
            got = C_root.cpu().numpy()
            a_rows = M if opA == "N" else K
            b_rows = K if opB == "N" else N
            tol = 3 * tolerance("f64", K, pr.A, a_rows, pr.B, b_rows, pr.beta, ref, M)
            err = float(np.abs(got[:, :M] - ref[:, :M]).max())
            pad_ok = bool(np.array_equal(got[:, M:], pr.C[:, M:]))
            ok = err <= tol
            if exact:  # sharded == oracle == single-GPU qgemm on the whole problem, bitwise
                C1 = torch.from_numpy(pr.C.copy()).to(dev)
                A1 = torch.from_numpy(pr.A).to(dev)
                for _ in range(2):
                    qg.qgemm(opA, opB, pr.alpha, A1, torch.from_numpy(pr.B).to(dev), pr.beta, C1,
                             M=M, N=N, K=K)
                single = C1.cpu().numpy()
                ok = (bool(np.array_equal(got[:, :M], ref[:, :M]))
                      and bool(np.array_equal(got[:, :M], single[:, :M])))
            q.put((ok, err, tol, pad_ok, qg.last_launch_count() > 0))
        dist.barrier()
        peer.close()
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("dist_kind", ["normal", "int8"])
@pytest.mark.parametrize("opA,opB,M,N,K", [("N", "H", 400, 300, 257), ("T", "N", 130, 70, 65)])
def test_p2p_epilogue_into_root_c_two_processes(opA, opB, M, N, K, dist_kind):
    """normal: within tolerance of the oracle; int8 (exact-integer inputs): the
    sharded result is bitwise equal to the oracle and to the single-GPU qgemm of
    the whole problem (SURVEY §8(e) invariant, T8)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, opA, opB, M, N, K, q, dist_kind))
             for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    ok, err, tol, pad_ok, launched = q.get(timeout=5)
    assert ok, (err, tol)
    assert pad_ok and launched
