"""B200-native quaternion GEMM (arXiv 1903.05575 hot path).

C <- alpha op(A) op(B) + beta C over Hamilton quaternions, op in {N, T, H},
column-major interleaved storage; FP64 on the FP64 tensor pipe (DMMA), FP32 as
3xTF32 on the tcgen05 tensor cores; small problems in one fused launch.  The computation lives in libqgemm.so (include/qgemm.h); this package is
the thin Python binding plus the multi-GPU row-block driver.
"""
from ._lib import EXPORTS, QgemmError, SO_PATH, load  # noqa: F401
from .qgemm import (  # noqa: F401
    get_workspace,
    host_workspace_bytes,
    last_launch_count,
    qgemm,
    qgemm_f32,
    qgemm_host,
    qgemm_ptr,
    ipc_handle,
    ipc_open,
    ipc_close,
    qgemm_naive,
    qherk,
    set_path_policy,
    PATH_AUTO,
    PATH_PACKED,
    PATH_SMALL,
    PATH_DIRECT,
    PATH_DIRECT32,
    PATH_SMALL_GENERAL,
    timing_collect,
    timing_enable,
    version,
    workspace_bytes,
    workspace_min_bytes,
)
