"""c1 latency probe: per-call time of small qgemm calls,
one call per graph replay and 32 calls back to back in one graph, next to a
trivial kernel; run it once per setting of QG_SMALL_PDL (read once per process).

    QG_SMALL_PDL=0 python tools/c1_probe.py ; QG_SMALL_PDL=1 python tools/c1_probe.py
    python tools/c1_probe.py --ncu N     # N plain c1 calls (for an ncu capture)
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_05575_b200 as qg  # noqa: E402
from tools.launch_floor import replay_seq_us, replay_us  # noqa: E402


def main():
    g = torch.Generator(device="cuda").manual_seed(0)
    if "--ncu" in sys.argv:
        n = int(sys.argv[sys.argv.index("--ncu") + 1])
        A = torch.randn(64, 64, 4, dtype=torch.float64, device="cuda", generator=g)
        B = torch.randn(64, 64, 4, dtype=torch.float64, device="cuda", generator=g)
        C = torch.zeros(64, 64, 4, dtype=torch.float64, device="cuda")
        for _ in range(n):
            qg.qgemm("N", "N", 1.0, A, B, 0.0, C)
        torch.cuda.synchronize()
        return
    x = torch.zeros(1, device="cuda")
    out = {"pdl": os.environ.get("QG_SMALL_PDL", "default"),
           "trivial_graph_us": replay_us(lambda: x.add_(1.0)),
           "trivial_seq32_us": replay_seq_us(lambda: x.add_(1.0))}
    print(json.dumps(out), flush=True)
    for M, N, K, beta in [(8, 8, 4, 0.0), (64, 64, 4, 0.0), (64, 64, 16, 0.0), (64, 64, 64, 0.0),
                          (64, 64, 64, 1.0), (128, 128, 128, 0.0), (256, 256, 256, 0.0)]:
        A = torch.randn(K, M, 4, dtype=torch.float64, device="cuda", generator=g)
        B = torch.randn(N, K, 4, dtype=torch.float64, device="cuda", generator=g)
        C = torch.randn(N, M, 4, dtype=torch.float64, device="cuda", generator=g)

        def call():
            qg.qgemm("N", "N", 1.0, A, B, beta, C)
        print(json.dumps({"M": M, "N": N, "K": K, "beta": beta, "graph_us": replay_us(call),
                          "seq32_us": replay_seq_us(call)}), flush=True)


if __name__ == "__main__":
    main()
