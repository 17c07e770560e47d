"""One c3-shaped qgemm call under a given path policy (ncu driver).

    python tools/prof_policy.py --policy 4 [--n 8192] [--ops NH]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_05575_b200 as qg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--policy", type=int, default=0)
ap.add_argument("--n", type=int, default=8192)
ap.add_argument("--k", type=int, default=None)
ap.add_argument("--ops", default="NH")
a = ap.parse_args()
qg.set_path_policy(a.policy)
g = torch.Generator(device="cuda").manual_seed(0)
n, K = a.n, a.k or a.n
ar, ac = (n, K) if a.ops[0] == "N" else (K, n)
br, bc = (K, n) if a.ops[1] == "N" else (n, K)
A = torch.randn((ac, ar, 4), dtype=torch.float64, device="cuda", generator=g)
B = torch.randn((bc, br, 4), dtype=torch.float64, device="cuda", generator=g)
C = torch.randn((n, n, 4), dtype=torch.float64, device="cuda", generator=g)
qg.qgemm(a.ops[0], a.ops[1], 1.0, A, B, 1.0, C, M=n, N=n, K=K)
torch.cuda.synchronize()
print("ok", float(C[0, 0, 0]))
