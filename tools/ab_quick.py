"""Quick A/B timing of the FP64 configs that matter for a kernel change: c3 (N/H
8192^3, beta = 1), c4 (32768^2 x 256, N/H, B == A, beta = 1), c2 NN (1024^3,
graph-replayed).  CUDA events, best of R calls.

    python tools/ab_quick.py [--reps 3]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_05575_b200 as qg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--policy", type=int, default=0)
a = ap.parse_args()
qg.set_path_policy(a.policy)
g = torch.Generator(device="cuda").manual_seed(0)


def best_ms(call, reps):
    call()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(reps):
        e0.record()
        call()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


out = {}
n = 8192
A = torch.randn((n, n, 4), dtype=torch.float64, device="cuda", generator=g)
B = torch.randn((n, n, 4), dtype=torch.float64, device="cuda", generator=g)
C = torch.randn((n, n, 4), dtype=torch.float64, device="cuda", generator=g)
ws = torch.empty(qg.workspace_bytes("N", "H", n, n, n), dtype=torch.uint8, device="cuda")
out["c3_ms"] = best_ms(lambda: qg.qgemm("N", "H", 1.0, A, B, 1.0, C, workspace=ws), a.reps)
out["c3_beta0_NN_ms"] = best_ms(lambda: qg.qgemm("N", "N", 1.0, A, B, 0.0, C, workspace=ws), a.reps)
del A, B, C, ws
n, K = 32768, 256
A = torch.rand((K, n, 4), dtype=torch.float64, device="cuda", generator=g)
C = torch.rand((n, n, 4), dtype=torch.float64, device="cuda", generator=g)
ws = torch.empty(qg.workspace_bytes("N", "H", n, n, K), dtype=torch.uint8, device="cuda")
out["c4_ms"] = best_ms(lambda: qg.qgemm("N", "H", 1.0, A, A, 1.0, C, M=n, N=n, K=K, workspace=ws), a.reps)
out["c4_herk_ms"] = best_ms(lambda: qg.qherk("L", "N", 1.0, A, 1.0, C, N=n), a.reps)
out["c4_beta0_ms"] = best_ms(lambda: qg.qgemm("N", "H", 1.0, A, A, 0.0, C, M=n, N=n, K=K, workspace=ws), a.reps)
del A, C, ws
n = 1024
A = torch.randn((n, n, 4), dtype=torch.float64, device="cuda", generator=g)
B = torch.randn((n, n, 4), dtype=torch.float64, device="cuda", generator=g)
C = torch.randn((n, n, 4), dtype=torch.float64, device="cuda", generator=g)
ws = torch.empty(max(256, qg.workspace_bytes("N", "N", n, n, n)), dtype=torch.uint8, device="cuda")
out["c2_NN_ms"] = best_ms(lambda: [qg.qgemm("N", "N", 0.75, A, B, -0.5, C, workspace=ws) for _ in range(20)],
                          a.reps) / 20
out["c2_beta0_NN_ms"] = best_ms(lambda: [qg.qgemm("N", "N", 0.75, A, B, 0.0, C, workspace=ws) for _ in range(20)],
                                a.reps) / 20
print(json.dumps(out))
