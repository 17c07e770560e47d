"""Crossover sweep: packed path vs one-launch small kernel (and, FP64, the direct path) (qgemm_set_path_policy).

Each call is captured once in a CUDA graph and replayed (host ctypes time is not
on the device timeline), CUDA events around the replays.

    python tools/small_sweep.py [--precision f64] [--out gpurun_out/small_sweep.jsonl]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_05575_b200 as qg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--precision", default="f64")
ap.add_argument("--out", default=None)
a = ap.parse_args()
dt = torch.float64 if a.precision == "f64" else torch.float32
fn = qg.qgemm if a.precision == "f64" else qg.qgemm_f32
g = torch.Generator(device="cuda").manual_seed(0)

SHAPES = [(n, n, n) for n in (16, 32, 64, 96, 128, 192, 256, 320, 384, 448, 512, 640, 768)]
SHAPES += [(64, 64, 4096), (4096, 64, 64), (64, 4096, 64), (256, 256, 1024), (1024, 1024, 16),
           (128, 128, 4096), (2048, 2048, 4), (64, 64, 8192), (32, 32, 32768), (4096, 4096, 2),
           (512, 512, 128), (128, 128, 2048)]


def graph_time(call, nrep=100):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        call()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=s):
            call()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    for _ in range(3):
        gr.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(nrep):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / nrep


out = open(a.out, "w") if a.out else None
for M, N, K in SHAPES:
    A = 2 * torch.rand((K, M, 4), dtype=dt, device="cuda", generator=g) - 1
    B = 2 * torch.rand((N, K, 4), dtype=dt, device="cuda", generator=g) - 1
    C = 2 * torch.rand((N, M, 4), dtype=dt, device="cuda", generator=g) - 1
    row = {"M": M, "N": N, "K": K, "dtype": a.precision}
    pols = (("packed", qg.PATH_PACKED), ("small", qg.PATH_SMALL))
    if a.precision == "f64":
        pols += (("direct", qg.PATH_DIRECT),)
    for name, pol in pols:
        old = qg.set_path_policy(pol)
        need = qg.workspace_bytes("N", "N", M, N, K, dt)
        ws = torch.empty(max(need, 256), dtype=torch.uint8, device="cuda")
        t = graph_time(lambda: fn("N", "N", 1.0, A, B, 1.0, C, M=M, N=N, K=K, workspace=ws))
        qg.set_path_policy(old)
        row[name + "_us"] = t * 1e3
        row[name + "_tflops"] = 32.0 * M * N * K / (t * 1e-3) / 1e12
    row["auto"] = "small" if qg.workspace_bytes("N", "N", M, N, K, dt) == 0 else "packed"
    print(json.dumps(row), flush=True)
    if out:
        out.write(json.dumps(row) + "\n")
