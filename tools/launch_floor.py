"""Floor of a one-kernel CUDA-graph replay on this box (context for c1's 6 us):
a trivial torch kernel vs the c1 qgemm call, both replayed back to back.

    python tools/launch_floor.py
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_05575_b200 as qg  # noqa: E402


def replay_us(call, nrep=2000):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        call()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            call()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    for _ in range(10):
        g.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(nrep):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / nrep * 1e3


x = torch.zeros(1, device="cuda")
A = torch.randn(64, 64, 4, dtype=torch.float64, device="cuda")
B = torch.randn(64, 64, 4, dtype=torch.float64, device="cuda")
C = torch.zeros(64, 64, 4, dtype=torch.float64, device="cuda")
out = {"trivial_kernel_graph_us": replay_us(lambda: x.add_(1.0)),
       "c1_qgemm_graph_us": replay_us(lambda: qg.qgemm("N", "N", 1.0, A, B, 0.0, C))}
print(json.dumps(out))


def replay_seq_us(call, n_in_graph=32, nrep=200):
    """Per-call time with n_in_graph calls captured back to back in one graph
    (graph-launch overhead amortised: kernel time + inter-kernel gap)."""
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        call()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(n_in_graph):
                call()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    for _ in range(5):
        g.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(nrep):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / (nrep * n_in_graph) * 1e3


out2 = {"trivial_kernel_seq32_us": replay_seq_us(lambda: x.add_(1.0)),
        "c1_qgemm_seq32_us": replay_seq_us(lambda: qg.qgemm("N", "N", 1.0, A, B, 0.0, C))}
print(json.dumps(out2))
