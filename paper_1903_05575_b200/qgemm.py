"""Python binding of the C ABI (same names as include/qgemm.h).

Tensors use the storage convention of the library: a CUDA tensor of shape
(ncols, ld, 4), C-contiguous, is a column-major quaternion matrix with leading
dimension ``ld`` (in quaternions) and interleaved components (PAPER.md
P:727-734).  This module only marshals pointers, sizes, the
current CUDA stream and a workspace; every step of the computation runs in the
kernels of libqgemm.so.
"""
from __future__ import annotations

import ctypes

import torch

from ._lib import QgemmError, load

# library-managed workspaces, one per (device, stream): calls on different
# streams may run concurrently and must not share scratch memory
_workspaces: dict[tuple[int, int], torch.Tensor] = {}


def _q4(x, dtype) -> ctypes.Array:
    """Quaternion scalar (real number or 4-sequence) -> host double[4]/float[4]."""
    vals = [0.0, 0.0, 0.0, 0.0]
    if isinstance(x, (int, float)):
        vals[0] = float(x)
    else:
        seq = [float(v) for v in (x.tolist() if hasattr(x, "tolist") else x)]
        vals[: len(seq)] = seq
    ct = ctypes.c_double if dtype == torch.float64 else ctypes.c_float
    return (ct * 4)(*vals)


def _ptr(t: torch.Tensor | None):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def leading_dim(t: torch.Tensor, name: str = "X") -> int:
    """Leading dimension (in quaternions) of a column-major (ncols, rows, 4) view.

    A contiguous tensor has ld = shape[1]; a row-block view of a larger matrix,
    X[:, r0:r1, :] (what the row-sharded driver hands each rank), keeps the
    parent's column stride, so ld = stride(0) / 4.  Anything else (a
    non-interleaved component stride, transposed or overlapping columns) is
    rejected: the kernels address element (i, j) at base + 4 (i + j ld)."""
    if t.dim() != 3 or t.shape[2] != 4:
        raise ValueError(f"{name}: expected an (ncols, rows, 4) tensor")
    if t.numel() == 0:  # nothing is addressed (strides of empty tensors are arbitrary)
        return max(1, t.shape[1])
    if t.stride(2) != 1 or (t.shape[1] > 1 and t.stride(1) != 4):
        raise ValueError(f"{name}: components and rows must be contiguous (strides (4 ld, 4, 1))")
    if t.shape[0] <= 1:
        return max(1, t.shape[1])
    s0 = t.stride(0)
    if s0 % 4 or s0 // 4 < t.shape[1]:
        raise ValueError(f"{name}: column stride {s0} is not 4 * ld with ld >= {t.shape[1]}")
    return s0 // 4


def _check(t: torch.Tensor, name: str, dtype):
    if t.dtype != dtype:
        raise TypeError(f"{name}: expected {dtype}, got {t.dtype}")
    if not t.is_cuda:
        raise TypeError(f"{name}: must be a CUDA tensor (no CPU path exists)")
    leading_dim(t, name)


def infer_dims(transA: str, transB: str, A: torch.Tensor, B: torch.Tensor, C: torch.Tensor):
    """(M, N, K) assuming no ld padding of C and A (explicit sizes override)."""
    M, N = C.shape[1], C.shape[0]
    K = A.shape[0] if transA.upper() == "N" else A.shape[1]
    return M, N, K


def workspace_bytes(transA: str, transB: str, M: int, N: int, K: int, dtype=torch.float64) -> int:
    return int(load().qgemm_workspace_bytes(transA.encode(), transB.encode(), M, N, K,
                                            0 if dtype == torch.float64 else 1))


def workspace_min_bytes(transA: str, transB: str, M: int, N: int, K: int, dtype=torch.float64) -> int:
    return int(load().qgemm_workspace_min_bytes(transA.encode(), transB.encode(), M, N, K,
                                                0 if dtype == torch.float64 else 1))


def get_workspace(nbytes: int, device, stream: torch.cuda.Stream | None = None) -> torch.Tensor:
    """Cached workspace of at least `nbytes` for calls on `stream` (default: the
    device's current stream).  It is allocated on that stream, so the caching
    allocator only recycles a replaced buffer after the stream's earlier work."""
    dev = torch.device(device)
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    st = stream or torch.cuda.current_stream(dev)
    key = (dev.index, st.cuda_stream)
    ws = _workspaces.get(key)
    if ws is None or ws.numel() < nbytes:
        _workspaces.pop(key, None)
        with torch.cuda.stream(st):
            ws = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=dev)
        _workspaces[key] = ws
    return ws


def _call(fn, name, transA, transB, M, N, K, alpha, A, B, beta, C, dtype, workspace, ws_bytes,
          stream):
    al, be = _q4(alpha, dtype), _q4(beta, dtype)
    lda = leading_dim(A, "A") if A is not None else 1
    ldb = leading_dim(B, "B") if B is not None else 1
    ldc = leading_dim(C, "C")
    args = [transA.encode(), transB.encode(), M, N, K, ctypes.cast(al, ctypes.c_void_p), _ptr(A),
            lda, _ptr(B), ldb, ctypes.cast(be, ctypes.c_void_p), _ptr(C), ldc]
    if workspace is not Ellipsis:
        args += [_ptr(workspace), ws_bytes]
    args += [ctypes.c_void_p(stream)]
    rc = fn(*args)
    if rc != 0:
        raise QgemmError(name, rc)
    return C


def qgemm(transA: str, transB: str, alpha, A: torch.Tensor, B: torch.Tensor, beta,
          C: torch.Tensor, M: int | None = None, N: int | None = None, K: int | None = None,
          workspace: torch.Tensor | None = None, stream: torch.cuda.Stream | None = None):
    """C <- alpha op(A) op(B) + beta C in FP64 (in place on C, asynchronous)."""
    return _qgemm_typed(load().qgemm, "qgemm", torch.float64, transA, transB, alpha, A, B, beta, C,
                        M, N, K, workspace, stream)


def qgemm_f32(transA: str, transB: str, alpha, A: torch.Tensor, B: torch.Tensor, beta,
              C: torch.Tensor, M: int | None = None, N: int | None = None, K: int | None = None,
              workspace: torch.Tensor | None = None, stream: torch.cuda.Stream | None = None):
    """FP32 variant: float storage, 3xTF32 products on the tcgen05 tensor cores with
    FP32 accumulation, or FP64 DMMA on the widened values in the
    one-launch small kernel; result rounded to FP32 once on store."""
    return _qgemm_typed(load().qgemm_f32, "qgemm_f32", torch.float32, transA, transB, alpha, A, B,
                        beta, C, M, N, K, workspace, stream)


def _qgemm_typed(fn, name, dtype, transA, transB, alpha, A, B, beta, C, M, N, K, workspace, stream):
    _check(C, "C", dtype)
    for t, nm in ((A, "A"), (B, "B")):
        if t is not None:
            _check(t, nm, dtype)
    m0, n0, k0 = infer_dims(transA, transB, A, B, C)
    M = m0 if M is None else M
    N = n0 if N is None else N
    K = k0 if K is None else K
    stream = stream or torch.cuda.current_stream(C.device)
    st = stream.cuda_stream
    need = workspace_bytes(transA, transB, M, N, K, dtype)
    if workspace is None:
        workspace = get_workspace(need, C.device, stream) if need else None
    nbytes = workspace.numel() * workspace.element_size() if workspace is not None else 0
    return _call(fn, name, transA, transB, M, N, K, alpha, A, B, beta, C, dtype, workspace, nbytes,
                 st)


def host_workspace_bytes(transA: str, transB: str, M: int, N: int, K: int,
                         dtype=torch.float64) -> int:
    return int(load().qgemm_host_workspace_bytes(transA.encode(), transB.encode(), M, N, K,
                                                 0 if dtype == torch.float64 else 1))


def qgemm_host(transA: str, transB: str, alpha, A: torch.Tensor, B: torch.Tensor, beta,
               C: torch.Tensor, M: int | None = None, N: int | None = None, K: int | None = None,
               workspace: torch.Tensor | None = None, device=None,
               stream: torch.cuda.Stream | None = None):
    """End-to-end QGEMM on HOST tensors (include/qgemm.h qgemm_host[_f32]): the
    library streams A/B/C through device staging (pin them for overlap) and
    writes the result back into the host C.  Asynchronous on `stream`; C is
    valid after the stream synchronises.  float64 -> qgemm_host, float32 ->
    qgemm_host_f32."""
    dtype = C.dtype
    if dtype not in (torch.float64, torch.float32):
        raise TypeError(f"C: expected float64/float32, got {dtype}")
    for t, nm in ((A, "A"), (B, "B"), (C, "C")):
        if t is None:
            continue
        if t.dtype != dtype:
            raise TypeError(f"{nm}: expected {dtype}, got {t.dtype}")
        if t.dim() != 3 or t.shape[2] != 4 or not t.is_contiguous():
            raise ValueError(f"{nm}: expected a contiguous (ncols, ld, 4) tensor")
    m0, n0, k0 = infer_dims(transA, transB, A, B, C)
    M = m0 if M is None else M
    N = n0 if N is None else N
    K = k0 if K is None else K
    dev = torch.device(device) if device is not None else torch.device("cuda",
                                                                       torch.cuda.current_device())
    stream = stream or torch.cuda.current_stream(dev)
    st = stream.cuda_stream
    need = host_workspace_bytes(transA, transB, M, N, K, dtype)
    if workspace is None:
        workspace = get_workspace(need, dev, stream) if need else None
    elif not workspace.is_cuda:
        raise TypeError("workspace: must be device memory")
    nbytes = workspace.numel() * workspace.element_size() if workspace is not None else 0
    fn = load().qgemm_host if dtype == torch.float64 else load().qgemm_host_f32
    return _call(fn, "qgemm_host", transA, transB, M, N, K, alpha, A, B, beta, C, dtype, workspace,
                 nbytes, st)


def qgemm_ptr(transA: str, transB: str, M: int, N: int, K: int, alpha, A: int, lda: int, B: int,
              ldb: int, beta, C: int, ldc: int, workspace: int, workspace_bytes: int, stream: int,
              dtype=torch.float64):
    """qgemm / qgemm_f32 on raw device addresses (ints): for operands that are not
    torch tensors of this process, e.g. root's C mapped with ipc_open()."""
    lib = load()
    fn = lib.qgemm if dtype == torch.float64 else lib.qgemm_f32
    al, be = _q4(alpha, dtype), _q4(beta, dtype)
    vp = ctypes.c_void_p
    rc = fn(transA.encode(), transB.encode(), M, N, K, ctypes.cast(al, vp), vp(A or None), lda,
            vp(B or None), ldb, ctypes.cast(be, vp), vp(C or None), ldc, vp(workspace or None),
            workspace_bytes, vp(stream))
    if rc != 0:
        raise QgemmError("qgemm", rc)


def ipc_handle(t: torch.Tensor) -> tuple[bytes, int, int]:
    """(64-byte CUDA IPC handle of the allocation holding t, byte offset of
    t.data_ptr() in it, allocation bytes)."""
    h = ctypes.create_string_buffer(64)
    off, size = ctypes.c_uint64(0), ctypes.c_uint64(0)
    rc = load().qgemm_ipc_handle(ctypes.c_void_p(t.data_ptr()), h, ctypes.byref(off),
                                 ctypes.byref(size))
    if rc != 0:
        raise QgemmError("qgemm_ipc_handle", rc)
    return h.raw, int(off.value), int(size.value)


def ipc_open(handle: bytes, offset: int) -> tuple[int, int]:
    """Map another process's allocation: (address of the shared tensor, mapping base)."""
    if len(handle) != 64:
        raise ValueError("IPC handle must be 64 bytes")
    p, b = ctypes.c_void_p(), ctypes.c_void_p()
    rc = load().qgemm_ipc_open(handle, offset, ctypes.byref(p), ctypes.byref(b))
    if rc != 0:
        raise QgemmError("qgemm_ipc_open", rc)
    return int(p.value), int(b.value)


def ipc_close(base: int) -> None:
    rc = load().qgemm_ipc_close(ctypes.c_void_p(base))
    if rc != 0:
        raise QgemmError("qgemm_ipc_close", rc)


def qgemm_naive(transA: str, transB: str, alpha, A: torch.Tensor, B: torch.Tensor, beta,
                C: torch.Tensor, M: int | None = None, N: int | None = None, K: int | None = None,
                stream: torch.cuda.Stream | None = None):
    """Debug path: one thread per output quaternion (not used by qgemm)."""
    _check(C, "C", torch.float64)
    m0, n0, k0 = infer_dims(transA, transB, A, B, C)
    M = m0 if M is None else M
    N = n0 if N is None else N
    K = k0 if K is None else K
    st = (stream or torch.cuda.current_stream(C.device)).cuda_stream
    return _call(load().qgemm_naive, "qgemm_naive", transA, transB, M, N, K, alpha, A, B, beta, C,
                 torch.float64, Ellipsis, 0, st)


def last_launch_count() -> int:
    return int(load().qgemm_last_launch_count())


HERK_ARGNAMES = {1: "uplo", 2: "trans", 3: "N", 4: "K", 6: "A", 7: "lda", 9: "C", 10: "ldc",
                 11: "workspace", 12: "workspace_bytes"}


def qherk(uplo: str, trans: str, alpha: float, A: torch.Tensor, beta: float, C: torch.Tensor,
          N: int | None = None, K: int | None = None, workspace: torch.Tensor | None = None,
          stream: torch.cuda.Stream | None = None):
    """FP64 Hermitian rank-K update on one triangle of C (include/qgemm.h qherk):
    trans 'N': C <- alpha A A^H + beta C (A stored N x K); 'H': C <- alpha A^H A + beta C."""
    _check(C, "C", torch.float64)
    _check(A, "A", torch.float64)
    N = C.shape[0] if N is None else N
    if K is None:
        K = A.shape[0] if trans.upper() == "N" else A.shape[1]
    stream = stream or torch.cuda.current_stream(C.device)
    st = stream.cuda_stream
    lib = load()
    need = int(lib.qherk_workspace_bytes(uplo.encode(), trans.encode(), N, K))
    if workspace is None:
        workspace = get_workspace(need, C.device, stream) if need else None
    nbytes = workspace.numel() * workspace.element_size() if workspace is not None else 0
    rc = lib.qherk(uplo.encode(), trans.encode(), N, K, float(alpha), _ptr(A), leading_dim(A, "A"),
                   float(beta), _ptr(C), leading_dim(C, "C"), _ptr(workspace), nbytes,
                   ctypes.c_void_p(st))
    if rc != 0:
        err = QgemmError("qherk", rc)
        if rc < 0:
            err.args = (f"qherk: argument {-rc} ({HERK_ARGNAMES.get(-rc, '?')}) invalid",)
        raise err
    return C


KINDS = ("pack", "mainloop", "scale", "naive", "small")

PATH_AUTO, PATH_PACKED, PATH_SMALL, PATH_DIRECT, PATH_DIRECT32, PATH_SMALL_GENERAL = 0, 1, 2, 3, 4, 5


def set_path_policy(policy: int) -> int:
    """0 auto, 1 always packed (pack launch + mainloop), 2 always the one-launch
    small kernel, 3 direct (FP64: persistent mainloop fed by TMA straight from
    the interleaved storage, no pack; FP32 packed), 4 direct with the 32-byte-
    swizzle tile feed only (3 and auto load the operands as 4-quaternion groups
    where M / N / K allow), 5 as 2 but never the tile-exact small kernel;
    returns the old one."""
    old = int(load().qgemm_set_path_policy(int(policy)))
    if old < 0:
        raise ValueError(f"invalid path policy {policy}")
    return old


def timing_enable(on: bool = True) -> None:
    """Bracket every library kernel launch of this thread with CUDA events."""
    load().qgemm_timing_enable(1 if on else 0)


def timing_collect() -> dict:
    """Synchronise on the recorded events; {kind: (total_ms, launches)}; clears."""
    ms = (ctypes.c_double * len(KINDS))()
    cnt = (ctypes.c_int * len(KINDS))()
    rc = load().qgemm_timing_collect(ms, cnt)
    if rc != 0:
        raise QgemmError("qgemm_timing_collect", rc)
    return {k: (ms[i], cnt[i]) for i, k in enumerate(KINDS)}


def version() -> str:
    return load().qgemm_version().decode()
