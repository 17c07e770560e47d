"""One c4-shaped qgemm call (M=N=32768, K=256, N/H, B == A) for ncu captures.

    python tools/prof_c4.py [--herk]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_05575_b200 as qg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--herk", action="store_true")
a = ap.parse_args()
g = torch.Generator(device="cuda").manual_seed(0)
n, K = 32768, 256
A = 2 * torch.rand((K, n, 4), dtype=torch.float64, device="cuda", generator=g) - 1
C = 2 * torch.rand((n, n, 4), dtype=torch.float64, device="cuda", generator=g) - 1
if a.herk:
    qg.qherk("L", "N", 1.0, A, 1.0, C)
else:
    qg.qgemm("N", "H", 1.0, A, A, 1.0, C, M=n, N=n, K=K)
torch.cuda.synchronize()
print("ok", float(C[0, 0, 0]))
