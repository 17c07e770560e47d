"""PAPER.md Fig. 4 on B200: wall time of QGEMM(N) vs
ZGEMM(2N) on the complex-block embedding (Eq. qmat_complex),
square, alpha = 1, beta = 0, FP64.  cuBLAS ZGEMM (torch.matmul
on complex128) stands in for MKL; cuBLAS DGEMM on the real-expanded shape
(4N x N x 4N, the same 32 N^3 real flops as QGEMM) is a second yardstick.
The paper's claim: QGEMM(N) ~2x faster than ZGEMM(2N).

    python tools/fig4_b200.py [--sizes 512,1024,2048,4096,8192]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_05575_b200 as qg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--sizes", default="64,128,256,384,512,768,1024,2048,3072,4096,6144,8192")
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
dev = torch.device("cuda")
g = torch.Generator(device="cuda").manual_seed(0)


def timeit(fn, reps):
    """Device time per call: the call is captured once in a CUDA graph and
    replayed (host-side Python/ctypes/dispatch cost is off the timeline for all
    three arms alike); best of `reps` batches of replays, CUDA events."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=s):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    gr.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    gr.replay()
    e1.record()
    torch.cuda.synchronize()
    nrep = max(1, min(200, int(50.0 / max(e0.elapsed_time(e1), 1e-3))))  # ~50 ms per batch
    best = 1e30
    for _ in range(reps):
        e0.record()
        for _ in range(nrep):
            gr.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / nrep)
    return best


for n in [int(s) for s in a.sizes.split(",")]:
    A = 2 * torch.rand((n, n, 4), dtype=torch.float64, device=dev, generator=g) - 1
    B = 2 * torch.rand((n, n, 4), dtype=torch.float64, device=dev, generator=g) - 1
    C = torch.empty((n, n, 4), dtype=torch.float64, device=dev)
    ws = qg.get_workspace(max(256, qg.workspace_bytes("N", "N", n, n, n)), dev)
    t_q = timeit(lambda: qg.qgemm("N", "N", 1.0, A, B, 0.0, C, workspace=ws), a.reps)
    del A, B, C
    Z1 = torch.randn((2 * n, 2 * n), dtype=torch.complex128, device=dev, generator=g)
    Z2 = torch.randn((2 * n, 2 * n), dtype=torch.complex128, device=dev, generator=g)
    t_z = timeit(lambda: torch.matmul(Z1, Z2), a.reps)
    del Z1, Z2
    D1 = torch.randn((4 * n, 4 * n), dtype=torch.float64, device=dev, generator=g)
    D2 = torch.randn((4 * n, n), dtype=torch.float64, device=dev, generator=g)
    t_d = timeit(lambda: torch.matmul(D1, D2), a.reps)
    del D1, D2
    torch.cuda.empty_cache()
    fl = 32.0 * n ** 3
    print(json.dumps({"N": n, "qgemm_ms": t_q, "zgemm_2N_ms": t_z, "dgemm_4NxNx4N_ms": t_d,
                      "zgemm_over_qgemm": t_z / t_q, "qgemm_tflops": fl / t_q / 1e9,
                      "zgemm_tflops_real": 2 * fl / t_z / 1e9, "dgemm_tflops": fl / t_d / 1e9}),
          flush=True)
