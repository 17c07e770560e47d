"""FP32 (3xTF32 tcgen05 pair kernel) throughput across square sizes, auto policy,
CUDA-graph replay: how much of the GPU the 256x128 pair tiles use below c3.

    python tools/f32_sizes.py
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_05575_b200 as qg  # noqa: E402


def graph_time(call, nrep=20):
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


g = torch.Generator(device="cuda").manual_seed(0)
for n in (512, 768, 1024, 1536, 2048, 3072, 4096, 6144):
    A = torch.randn((n, n, 4), dtype=torch.float32, device="cuda", generator=g)
    B = torch.randn((n, n, 4), dtype=torch.float32, device="cuda", generator=g)
    C = torch.randn((n, n, 4), dtype=torch.float32, device="cuda", generator=g)
    ws = torch.empty(max(256, qg.workspace_bytes("N", "H", n, n, n, torch.float32)), dtype=torch.uint8,
                     device="cuda")
    t = graph_time(lambda: qg.qgemm_f32("N", "H", 1.0, A, B, 1.0, C, workspace=ws))
    pairs = -(-n // 256) * -(-n // 128)
    print(json.dumps({"n": n, "ms": t, "tflops": 32.0 * n ** 3 / (t * 1e-3) / 1e12, "pair_tiles": pairs,
                      "waves_of_74": pairs / 74}), flush=True)
    del A, B, C, ws
