"""ctypes binding of libqgemm.so (include/qgemm.h).  Argument marshalling only.

The product path has no fallback: if the shared library is missing or fails
to load, every entry point raises.
"""
from __future__ import annotations

import ctypes
import os

PKG = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(PKG, "libqgemm.so")

#: every symbol include/qgemm.h declares
EXPORTS = ("qgemm", "qgemm_f32", "qgemm_workspace_bytes", "qgemm_workspace_min_bytes",
           "qgemm_naive", "qherk", "qherk_workspace_bytes", "qgemm_last_launch_count",
           "qgemm_set_path_policy", "qgemm_host", "qgemm_host_f32", "qgemm_host_workspace_bytes",
           "qgemm_ipc_handle", "qgemm_ipc_open", "qgemm_ipc_close",
           "qgemm_timing_enable", "qgemm_timing_collect", "qgemm_version", "qgemm_pack_panel")

_lib = None


class QgemmError(RuntimeError):
    """Non-zero return of a C-ABI call (-i: argument i invalid; >0: cudaError_t)."""

    ARGNAMES = {1: "transA", 2: "transB", 3: "M", 4: "N", 5: "K", 6: "alpha", 7: "A", 8: "lda",
                9: "B", 10: "ldb", 11: "beta", 12: "C", 13: "ldc", 14: "workspace",
                15: "workspace_bytes", 16: "stream"}

    def __init__(self, fn: str, code: int):
        self.code = code
        if code < 0:
            msg = f"{fn}: argument {-code} ({self.ARGNAMES.get(-code, '?')}) invalid"
        else:
            msg = f"{fn}: CUDA error {code}"
        super().__init__(msg)


def load():
    """Load libqgemm.so (raises OSError/FileNotFoundError loudly if absent)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(SO_PATH):
        raise FileNotFoundError(
            f"{SO_PATH} not built: run `python -m paper_1903_05575_b200.build` "
            "(no CPU fallback exists)")
    lib = ctypes.CDLL(SO_PATH)
    c, i64, vp, sz = ctypes.c_char, ctypes.c_int64, ctypes.c_void_p, ctypes.c_size_t
    common = [c, c, i64, i64, i64, vp, vp, i64, vp, i64, vp, vp, i64]
    lib.qgemm.argtypes = common + [vp, sz, vp]
    lib.qgemm.restype = ctypes.c_int
    lib.qgemm_f32.argtypes = common + [vp, sz, vp]
    lib.qgemm_f32.restype = ctypes.c_int
    lib.qgemm_host.argtypes = common + [vp, sz, vp]
    lib.qgemm_host.restype = ctypes.c_int
    lib.qgemm_host_f32.argtypes = common + [vp, sz, vp]
    lib.qgemm_host_f32.restype = ctypes.c_int
    lib.qgemm_host_workspace_bytes.argtypes = [c, c, i64, i64, i64, ctypes.c_int]
    lib.qgemm_host_workspace_bytes.restype = sz
    u64p = ctypes.POINTER(ctypes.c_uint64)
    lib.qgemm_ipc_handle.argtypes = [vp, ctypes.c_char_p, u64p, u64p]
    lib.qgemm_ipc_handle.restype = ctypes.c_int
    lib.qgemm_ipc_open.argtypes = [ctypes.c_char_p, ctypes.c_uint64, ctypes.POINTER(vp),
                                   ctypes.POINTER(vp)]
    lib.qgemm_ipc_open.restype = ctypes.c_int
    lib.qgemm_ipc_close.argtypes = [vp]
    lib.qgemm_ipc_close.restype = ctypes.c_int
    lib.qgemm_naive.argtypes = common + [vp]
    lib.qgemm_naive.restype = ctypes.c_int
    lib.qgemm_workspace_bytes.argtypes = [c, c, i64, i64, i64, ctypes.c_int]
    lib.qgemm_workspace_bytes.restype = sz
    lib.qgemm_workspace_min_bytes.argtypes = [c, c, i64, i64, i64, ctypes.c_int]
    lib.qgemm_workspace_min_bytes.restype = sz
    lib.qgemm_last_launch_count.restype = ctypes.c_int
    lib.qgemm_set_path_policy.argtypes = [ctypes.c_int]
    lib.qgemm_set_path_policy.restype = ctypes.c_int
    lib.qgemm_version.restype = ctypes.c_char_p
    dbl = ctypes.c_double
    lib.qherk.argtypes = [c, c, i64, i64, dbl, vp, i64, dbl, vp, i64, vp, sz, vp]
    lib.qherk.restype = ctypes.c_int
    lib.qherk_workspace_bytes.argtypes = [c, c, i64, i64]
    lib.qherk_workspace_bytes.restype = sz
    lib.qgemm_pack_panel.argtypes = [c, ctypes.c_int, i64, i64, vp, i64, vp, sz, vp]
    lib.qgemm_pack_panel.restype = ctypes.c_int
    lib.qgemm_timing_enable.argtypes = [ctypes.c_int]
    lib.qgemm_timing_enable.restype = None
    lib.qgemm_timing_collect.argtypes = [ctypes.POINTER(ctypes.c_double),
                                         ctypes.POINTER(ctypes.c_int)]
    lib.qgemm_timing_collect.restype = ctypes.c_int
    _lib = lib
    return lib
