"""c4 with beta = 1 vs beta = 0 (no C read in the epilogue) vs alpha = 0 style
store-only: how much of c4's time the epilogue's C read costs.

    python tools/c4_beta_probe.py
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_05575_b200 as qg  # noqa: E402

n, K = 32768, 256
g = torch.Generator(device="cuda").manual_seed(0)
A = torch.rand((K, n, 4), dtype=torch.float64, device="cuda", generator=g)
C = torch.rand((n, n, 4), dtype=torch.float64, device="cuda", generator=g)
ws = torch.empty(qg.workspace_bytes("N", "H", n, n, K), dtype=torch.uint8, device="cuda")
out = {}
for pol_name, pol in (("auto", qg.PATH_AUTO), ("direct", qg.PATH_DIRECT)):
    old = qg.set_path_policy(pol)
    for beta in (1.0, 0.0):
        for _ in range(2):
            qg.qgemm("N", "H", 1.0, A, A, beta, C, M=n, N=n, K=K, workspace=ws)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e30
        for _ in range(6):
            e0.record()
            qg.qgemm("N", "H", 1.0, A, A, beta, C, M=n, N=n, K=K, workspace=ws)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        out[f"{pol_name}_beta{int(beta)}_ms"] = best
        out[f"{pol_name}_beta{int(beta)}_tflops"] = 32.0 * n * n * K / (best * 1e-3) / 1e12
    qg.set_path_policy(old)
print(json.dumps(out))
