"""Per-call time of small qgemm calls with 32 calls captured back to back in one
CUDA graph (graph-launch overhead amortised): how c1's time splits into a fixed
part and a K-dependent part.

    python tools/small_latency.py
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_05575_b200 as qg  # noqa: E402
from tools.launch_floor import replay_seq_us  # noqa: E402

g = torch.Generator(device="cuda").manual_seed(0)
for M, N, K, beta in [(8, 8, 4, 0.0), (64, 64, 4, 0.0), (64, 64, 16, 0.0), (64, 64, 64, 0.0),
                      (64, 64, 64, 1.0), (64, 64, 256, 0.0), (128, 128, 128, 0.0), (256, 256, 256, 0.0)]:
    A = torch.randn(K, M, 4, dtype=torch.float64, device="cuda", generator=g)
    B = torch.randn(N, K, 4, dtype=torch.float64, device="cuda", generator=g)
    C = torch.randn(N, M, 4, dtype=torch.float64, device="cuda", generator=g)
    us = replay_seq_us(lambda: qg.qgemm("N", "N", 1.0, A, B, beta, C))
    print(json.dumps({"M": M, "N": N, "K": K, "beta": beta, "seq32_us": us}), flush=True)
