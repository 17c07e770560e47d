"""Floor of a one-kernel CUDA-graph replay on this box (context for c1's time):
a trivial torch kernel vs the c1 qgemm call, each replayed back to back as a
one-call graph, and per call with 32 calls captured in one graph (graph-launch
overhead amortised: kernel time + inter-kernel gap).

    python tools/launch_floor.py
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_05575_b200 as qg  # noqa: E402


def _capture(call, n_in_graph):
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
    return g


def _us_per_replay(g, nrep):
    for _ in range(10):
        g.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(nrep):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / nrep * 1e3


def replay_us(call, nrep=2000):
    """Microseconds per replay of a one-call graph."""
    return _us_per_replay(_capture(call, 1), nrep)


def replay_seq_us(call, n_in_graph=32, nrep=200):
    """Microseconds per call with n_in_graph calls back to back in one graph."""
    return _us_per_replay(_capture(call, n_in_graph), nrep) / n_in_graph


def main():
    x = torch.zeros(1, device="cuda")
    A = torch.randn(64, 64, 4, dtype=torch.float64, device="cuda")
    B = torch.randn(64, 64, 4, dtype=torch.float64, device="cuda")
    C = torch.zeros(64, 64, 4, dtype=torch.float64, device="cuda")

    def c1():
        qg.qgemm("N", "N", 1.0, A, B, 0.0, C)

    print(json.dumps({"trivial_kernel_graph_us": replay_us(lambda: x.add_(1.0)),
                      "c1_qgemm_graph_us": replay_us(c1),
                      "trivial_kernel_seq32_us": replay_seq_us(lambda: x.add_(1.0)),
                      "c1_qgemm_seq32_us": replay_seq_us(c1)}))


if __name__ == "__main__":
    main()
