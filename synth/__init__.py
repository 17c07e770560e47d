"""Seeded synthetic inputs shared by tests/, bench.py and smoke().

This package holds NO quaternion-GEMM arithmetic: it only draws numbers and
lays them out in the column-major interleaved storage of the C ABI.  It is the
one module both the oracle side and the CUDA side may use (task rule ③).
"""
from .inputs import (  # noqa: F401
    CONFIGS,
    Problem,
    make_problem,
    quat_matrix,
    hermitian_matrix,
    counter_uniform,
    stored_shape,
)
