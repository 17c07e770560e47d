"""c4 timing (qgemm N/H with B == A, and qherk), device-resident, CUDA events;
for A/B builds of epilogue knobs.

    python tools/c4_time.py [--n 32768] [--k 256]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_05575_b200 as qg  # noqa: E402


def timed(fn, reps=3, warm=1):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=32768)
    ap.add_argument("--k", type=int, default=256)
    ap.add_argument("--tag", default="")
    a = ap.parse_args()
    g = torch.Generator(device="cuda").manual_seed(0)
    A = 2 * torch.rand((a.k, a.n, 4), dtype=torch.float64, device="cuda", generator=g) - 1
    C = 2 * torch.rand((a.n, a.n, 4), dtype=torch.float64, device="cuda", generator=g) - 1
    fl = 32.0 * a.n * a.n * a.k
    ms = timed(lambda: qg.qgemm("N", "H", 1.0, A, A, 1.0, C, M=a.n, N=a.n, K=a.k))
    ms0 = timed(lambda: qg.qgemm("N", "H", 1.0, A, A, 0.0, C, M=a.n, N=a.n, K=a.k))
    mh = timed(lambda: qg.qherk("L", "N", 1.0, A, 1.0, C))
    print(json.dumps({"tag": a.tag, "n": a.n, "k": a.k, "qgemm_ms": ms, "qgemm_tflops": fl / ms / 1e9,
                      "qgemm_beta0_ms": ms0, "qherk_ms": mh}), flush=True)


if __name__ == "__main__":
    main()
