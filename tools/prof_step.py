"""One qgemm call at bench size for ncu captures (pack A, pack B, mainloop).

    python tools/prof_step.py [--n 8192] [--precision f64] [--ops NH]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_05575_b200 as qg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=8192)
ap.add_argument("--precision", default="f64")
ap.add_argument("--ops", default="NH")
ap.add_argument("--reps", type=int, default=1)
a = ap.parse_args()
dt = torch.float64 if a.precision == "f64" else torch.float32
g = torch.Generator(device="cuda").manual_seed(0)
n = a.n
A = torch.randn((n, n, 4), dtype=dt, device="cuda", generator=g)
B = torch.randn((n, n, 4), dtype=dt, device="cuda", generator=g)
C = torch.randn((n, n, 4), dtype=dt, device="cuda", generator=g)
fn = qg.qgemm if a.precision == "f64" else qg.qgemm_f32
for _ in range(a.reps):
    fn(a.ops[0], a.ops[1], 1.0, A, B, 1.0, C)
torch.cuda.synchronize()
print("ok", float(C[0, 0, 0]))
