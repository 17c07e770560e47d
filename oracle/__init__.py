"""CPU correctness oracle for quaternion GEMM (arXiv 1903.05575).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / ``--impl reference`` legs of bench.py.  The product package
``paper_1903_05575_b200`` never imports it, and it never imports the product.

Pinned functions (tests/test_oracle_pins.py): hmul, hconj, qgemm, qgemm_entries,
qgemv, chi (complex embedding).  No function here is "parity unpinned".
"""
from .oracle import (  # noqa: F401
    build_oracle,
    hmul,
    hconj,
    qgemm,
    qgemm_entries,
    qgemv,
    max_threads,
    lib_path,
)
from .embedding import chi, unchi, op_materialise  # noqa: F401
