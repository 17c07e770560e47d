"""Packed (pack launch + mainloop) vs TMA-fed FP64 mainloop across shapes:
(4-quaternion-group and 32-byte-only tiles): the data behind the auto policy's choice.  CUDA-graph replay,
CUDA events.

    python tools/feed_sweep.py [--out gpurun_out/feed_sweep.jsonl]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_05575_b200 as qg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--out", default=None)
ap.add_argument("--small-shapes", action="store_true", help="the small/direct/packed crossover region")
a = ap.parse_args()
g = torch.Generator(device="cuda").manual_seed(0)
SHAPES = [(n, n, n, ops) for n in (384, 512, 768, 1024, 1536, 2048, 3072, 4096) for ops in ("NN", "NH", "TN", "TH")]
SHAPES += [(8192, 8192, 256, "NH"), (4096, 4096, 256, "NH"), (2048, 2048, 8192, "NH"), (4096, 4096, 1024, "NH")]
if a.small_shapes:
    SHAPES = [(n, n, n, ops) for n in (128, 192, 256, 320, 384, 448, 512) for ops in ("NN", "TN")]


def graph_time(call):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        call()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=s):
            call()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    gr.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    gr.replay()
    e1.record()
    torch.cuda.synchronize()
    nrep = max(3, min(100, int(100.0 / max(e0.elapsed_time(e1), 1e-3))))
    best = 1e30
    for _ in range(3):
        e0.record()
        for _ in range(nrep):
            gr.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / nrep)
    return best


out = open(a.out, "w") if a.out else None
for M, N, K, ops in SHAPES:
    ar, ac = (M, K) if ops[0] == "N" else (K, M)
    br, bc = (K, N) if ops[1] == "N" else (N, K)
    A = torch.randn((ac, ar, 4), dtype=torch.float64, device="cuda", generator=g)
    B = torch.randn((bc, br, 4), dtype=torch.float64, device="cuda", generator=g)
    C = torch.randn((N, M, 4), dtype=torch.float64, device="cuda", generator=g)
    row = {"M": M, "N": N, "K": K, "ops": ops}
    pols = (("packed", qg.PATH_PACKED), ("tma", qg.PATH_DIRECT), ("tma32", qg.PATH_DIRECT32))
    if a.small_shapes:
        pols += (("small", qg.PATH_SMALL),)
    for name, pol in pols:
        old = qg.set_path_policy(pol)
        ws = torch.empty(max(256, qg.workspace_bytes(ops[0], ops[1], M, N, K)), dtype=torch.uint8, device="cuda")
        t = graph_time(lambda: qg.qgemm(ops[0], ops[1], 1.0, A, B, 1.0, C, M=M, N=N, K=K, workspace=ws))
        qg.set_path_policy(old)
        row[name + "_ms"] = t
        row[name + "_tflops"] = 32.0 * M * N * K / (t * 1e-3) / 1e12
        del ws
    row["tma_over_packed"] = row["packed_ms"] / row["tma_ms"]
    row["tma_over_tma32"] = row["tma32_ms"] / row["tma_ms"]
    print(json.dumps(row), flush=True)
    if out:
        out.write(json.dumps(row) + "\n")
    del A, B, C
    torch.cuda.empty_cache()
