"""c3 FP32 (8192^3 N/H, alpha = beta = 1) and two smaller squares: CUDA events, W warm-up
calls, then the mean of R back-to-back calls and the best single call (A/B of FP32 kernel
knobs; the clock under the power cap decides, so compare runs on one box, interleaved).

    python tools/f32_c3_time.py [--reps 10]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_05575_b200 as qg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=10)
a = ap.parse_args()
g = torch.Generator(device="cuda").manual_seed(0)
out = {}
for n in (8192, 4096, 2048):
    A = torch.randn((n, n, 4), dtype=torch.float32, device="cuda", generator=g)
    B = torch.randn((n, n, 4), dtype=torch.float32, device="cuda", generator=g)
    C = torch.zeros((n, n, 4), dtype=torch.float32, device="cuda")
    ws = qg.get_workspace(qg.workspace_bytes("N", "H", n, n, n, torch.float32), torch.device("cuda"))
    call = lambda: qg.qgemm_f32("N", "H", 1.0, A, B, 1.0, C, workspace=ws)  # noqa: E731
    for _ in range(3):
        call()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(a.reps + 1)]
    ev[0].record()
    for i in range(a.reps):
        call()
        ev[i + 1].record()
    torch.cuda.synchronize()
    ts = [ev[i].elapsed_time(ev[i + 1]) for i in range(a.reps)]
    out[f"n{n}_mean_ms"] = sum(ts) / len(ts)
    out[f"n{n}_best_ms"] = min(ts)
    out[f"n{n}_tflops_mean"] = 32.0 * n ** 3 / (sum(ts) / len(ts) * 1e-3) / 1e12
    del A, B, C
print(json.dumps(out))
