"""One c4-shaped qgemm call (M=N=32768, K=256, N/H, B == A) for ncu captures.

    python tools/prof_c4.py [--herk] [--beta B]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_05575_b200 as qg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--herk", action="store_true")
ap.add_argument("--beta", type=float, default=1.0)
ap.add_argument("--ldc-pad", type=int, default=0, help="C leading dimension = n + pad")
ap.add_argument("--time", action="store_true", help="time 3 calls (CUDA events) instead of one")
a = ap.parse_args()
g = torch.Generator(device="cuda").manual_seed(0)
n, K = 32768, 256
A = 2 * torch.rand((K, n, 4), dtype=torch.float64, device="cuda", generator=g) - 1
C = 2 * torch.rand((n, n + a.ldc_pad, 4), dtype=torch.float64, device="cuda", generator=g) - 1


def call():
    if a.herk:
        qg.qherk("L", "N", 1.0, A, a.beta, C, N=n)
    else:
        qg.qgemm("N", "H", 1.0, A, A, a.beta, C, M=n, N=n, K=K)


call()
torch.cuda.synchronize()
if a.time:
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(3):
        e0.record()
        call()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print("ms", best, "tflops", 32.0 * n * n * K / (best * 1e-3) / 1e12 / (2 if a.herk else 1))
print("ok", float(C[0, 0, 0]))
