"""Row-block multi-GPU driver (north star item (4)).

C <- alpha op(A) op(B) + beta C with C sharded by row blocks over the ranks of
a process group (one process per GPU, NCCL over NVLink 5 / NVSwitch):

  * rank r owns rows [r0, r1) of C and op(A): C_r = alpha op(A)_r op(B) + beta C_r,
    an independent QGEMM of shape (r1 - r0) x N x K -- the sharded unit;
  * op(B) is needed by every rank: ONE exchange step, `broadcast` of B's storage
    from `root` (skipped with broadcast_b=False when B is already resident);
  * ONE collection step: every rank sends its compact C_r (ld = r1 - r0) to
    `root`, which copies it into the row block of the column-major full C
    (ldc = M): the relayout of a strided row block.

Fused collection (qgemm_rowsharded_p2p, the default of bench.py at N > 1): C
lives on root only.  Root's C allocation is mapped into every rank once
(PeerC: CUDA IPC handle + offset, include/qgemm.h "Peer memory"), and each
rank's qgemm writes its finished tiles straight into root's C over NVLink /
NVSwitch (C argument = root's C + r0 rows, ldc = root's leading dimension):
the collection overlaps the mainloop tile by tile and neither a gather nor a
relayout pass exists.  A one-element all_reduce after the local QGEMM is the
completion barrier (stream-ordered, so root's later work sees every row block).

Row split: rows_for_rank() -- contiguous blocks, sizes differ by at most one
64-row tile so every rank's mainloop tiles are full except the global tail.
The local GEMM is libqgemm.so's qgemm (no CPU path); tests on CPU/gloo inject
the oracle through `local_gemm` to exercise this host logic only.
"""
from __future__ import annotations

from typing import Callable

import torch
import torch.distributed as dist

TILE = 64


def _ld(t: torch.Tensor, name: str) -> int:
    """Leading dimension of a (ncols, rows, 4) view (qgemm.leading_dim; no CUDA needed)."""
    from .qgemm import leading_dim
    return leading_dim(t, name)


def rows_for_rank(M: int, world: int, rank: int, tile: int = TILE) -> tuple[int, int]:
    """[r0, r1) of the row block of `rank`: whole tiles split as evenly as possible."""
    tiles = (M + tile - 1) // tile
    base, extra = divmod(tiles, world)
    t0 = rank * base + min(rank, extra)
    t1 = t0 + base + (1 if rank < extra else 0)
    return min(M, t0 * tile), min(M, t1 * tile)


def qgemm_rowsharded(transA: str, transB: str, alpha, A_local: torch.Tensor, B: torch.Tensor,
                     beta, C_local: torch.Tensor, M: int, N: int, K: int,
                     group=None, root: int = 0, broadcast_b: bool = True,
                     gather: bool = True, C_full: torch.Tensor | None = None,
                     local_gemm: Callable | None = None):
    """Sharded QGEMM step: broadcast B (from root) -> local QGEMM -> gather C.

    A_local: stored operand whose op() is rows [r0, r1) of op(A):
             opA = 'N': (K, M_loc, 4) with ld = M_loc; opA = 'T'/'H': (M_loc, K, 4).
    B:       full stored B on every rank (contents only meaningful on root when
             broadcast_b=True); shape (ncols, ldb, 4).
    C_local: (N, M_loc, 4), this rank's rows of C (compact, ld = M_loc).
    C_full:  on root when gather=True: (N, ldc >= M, 4) receiving all row blocks.
    Returns C_full on root (gather=True), else C_local.
    """
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    r0, r1 = rows_for_rank(M, world, rank)
    m_loc = r1 - r0
    assert C_local.shape[0] == N and C_local.shape[1] >= m_loc  # empty shard allowed
    if broadcast_b:
        dist.broadcast(B, src=root, group=group)
    if local_gemm is None:
        from .qgemm import qgemm as local_gemm_fn  # libqgemm.so, no fallback
        local_gemm = local_gemm_fn
    if m_loc > 0:
        local_gemm(transA, transB, alpha, A_local, B, beta, C_local, M=m_loc, N=N, K=K)
    if not gather:
        return C_local
    # gloo moves host memory only: CUDA tensors are staged through the host
    # there (bench.py --debug-one-device); NCCL sends device memory directly
    host_stage = C_local.is_cuda and dist.get_backend(group) == "gloo"
    if rank == root:
        assert C_full is not None and C_full.shape[0] == N and C_full.shape[1] >= M
        C_full[:, r0:r1, :].copy_(C_local[:, :m_loc, :])
        bufs = []
        ops = []
        for src in range(world):
            if src == root:
                continue
            s0, s1 = rows_for_rank(M, world, src)
            if s1 == s0:
                continue
            buf = torch.empty((N, s1 - s0, 4), dtype=C_local.dtype,
                              device="cpu" if host_stage else C_local.device)
            bufs.append((s0, s1, buf))
            ops.append(dist.P2POp(dist.irecv, buf, src, group))
        for w in dist.batch_isend_irecv(ops) if ops else []:
            w.wait()
        for s0, s1, buf in bufs:  # relayout: compact C_r -> strided row block of C
            C_full[:, s0:s1, :].copy_(buf)
        return C_full
    if m_loc > 0:
        send = C_local if C_local.shape[1] == m_loc else C_local[:, :m_loc, :].contiguous()
        if host_stage:
            send = send.cpu()
        for w in dist.batch_isend_irecv([dist.P2POp(dist.isend, send, root, group)]):
            w.wait()
    return C_local


class PeerC:
    """Root's column-major C (N columns, leading dimension ldc >= M) mapped into
    the address space of every rank of `group` (created once, reused per step).

    Root passes its C tensor; the other ranks pass None.  `share`/`open_` map a
    tensor to a picklable token and back to an address; the defaults are the
    library's CUDA IPC calls (qgemm_ipc_handle / qgemm_ipc_open), the CPU tests
    inject shared-memory files."""

    def __init__(self, C_full: torch.Tensor | None, group=None, root: int = 0,
                 share: Callable | None = None, open_: Callable | None = None,
                 close: Callable | None = None):
        from .qgemm import ipc_close, ipc_handle, ipc_open
        self.group, self.root = group, root
        rank = dist.get_rank(group)
        share = share or (lambda t: ipc_handle(t)[:2])
        open_ = open_ or ipc_open
        self._close = close or ipc_close
        info = [None]
        if rank == root:
            assert C_full is not None and C_full.dim() == 3 and C_full.shape[2] == 4
            assert C_full.is_contiguous()
            info[0] = (share(C_full), int(C_full.shape[0]), int(C_full.shape[1]),
                       str(C_full.dtype), C_full.element_size())
        dist.broadcast_object_list(info, src=root, group=group)
        token, self.ncols, self.ldc, self.dtype_name, self.elsize = info[0]
        if rank == root:
            self.addr, self.base, self.tensor = C_full.data_ptr(), None, C_full
        else:
            self.addr, self.base = open_(*token) if isinstance(token, tuple) else open_(token)
            self.tensor = None

    def row_addr(self, r0: int) -> int:
        """Address of C(r0, 0) (column-major, 4 scalars per quaternion)."""
        return self.addr + 4 * self.elsize * r0

    def close(self):
        if self.base is not None:
            self._close(self.base)
            self.base = None


def qgemm_rowsharded_p2p(transA: str, transB: str, alpha, A_local: torch.Tensor, B: torch.Tensor,
                         beta, peer: PeerC, M: int, N: int, K: int, group=None, root: int = 0,
                         broadcast_b: bool = True, workspace: torch.Tensor | None = None,
                         local_gemm_ptr: Callable | None = None, barrier: bool = True):
    """Sharded QGEMM step with the collection fused into the epilogue:
    broadcast B (NCCL) -> local QGEMM whose epilogue stores into root's C over
    peer memory -> completion all_reduce.  A_local as qgemm_rowsharded; root's
    C (PeerC) is read (beta != 0) and written in place; returns None."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    r0, r1 = rows_for_rank(M, world, rank)
    m_loc = r1 - r0
    assert peer.ncols == N and peer.ldc >= M
    if broadcast_b:
        dist.broadcast(B, src=root, group=group)
    else:
        # peers read (beta != 0) and write root's C: order them after root's
        # earlier work on C (the broadcast does that when it runs)
        flag = torch.zeros(1, dtype=torch.float32, device=A_local.device)
        dist.all_reduce(flag, group=group)
    if m_loc > 0:
        # A_local may be a row-block view of a larger stored A (c4: rows
        # [r0, r1) of the broadcast A, lda = M): ld from the strides, not the shape
        lda, ldb = _ld(A_local, "A_local"), _ld(B, "B")
        if local_gemm_ptr is None:
            from .qgemm import get_workspace, qgemm_ptr, workspace_bytes
            dt = A_local.dtype
            need = workspace_bytes(transA, transB, m_loc, N, K, dt)
            ws = workspace
            cur = torch.cuda.current_stream(A_local.device)
            if ws is None or ws.numel() * ws.element_size() < need:
                ws = get_workspace(need, A_local.device, cur) if need else None
            st = cur.cuda_stream
            qgemm_ptr(transA, transB, m_loc, N, K, alpha, A_local.data_ptr(), lda, B.data_ptr(),
                      ldb, beta, peer.row_addr(r0), peer.ldc,
                      ws.data_ptr() if ws is not None else 0,
                      ws.numel() * ws.element_size() if ws is not None else 0, st, dtype=dt)
        else:
            local_gemm_ptr(transA, transB, m_loc, N, K, alpha, A_local, lda, B, ldb, beta,
                           peer.row_addr(r0), peer.ldc)
    if barrier:
        flag = torch.zeros(1, dtype=torch.float32, device=A_local.device)
        dist.all_reduce(flag, group=group)
