"""Where the time of one c3 qgemm_host call goes: wall time of the call on its
stream (CUDA events) vs the summed durations of the kernels it launched
(qgemm_timing_*), i.e. how much of the PCIe traffic is not hidden.

    python tools/host_timeline.py [--n 8192]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_05575_b200 as qg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=8192)
a = ap.parse_args()
n = a.n
rng = np.random.default_rng(0)
A, B, C = (torch.from_numpy(rng.standard_normal((n, n, 4))).pin_memory() for _ in range(3))
ws = torch.empty(qg.host_workspace_bytes("N", "H", n, n, n), dtype=torch.uint8, device="cuda")
qg.qgemm_host("N", "H", 1.0, A, B, 1.0, C, workspace=ws)
torch.cuda.synchronize()
rows = []
for _ in range(3):
    qg.timing_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    qg.qgemm_host("N", "H", 1.0, A, B, 1.0, C, workspace=ws)
    e1.record()
    torch.cuda.synchronize()
    kt = qg.timing_collect()
    qg.timing_enable(False)
    wall = e0.elapsed_time(e1)
    kern = sum(v[0] for v in kt.values())
    rows.append({"wall_ms": wall, "kernel_ms": kern, "exposed_ms": wall - kern,
                 "per_kind": {k: {"ms": v[0], "launches": v[1]} for k, v in kt.items() if v[1]}})
print(json.dumps(rows[-1]))
