"""Per-CTA phase timeline of the persistent DMMA kernel (diagnostic build with
-DQG_TRACE copied over libqgemm.so; see qg_dmma.cuh QG_TR): where a call's time
goes between the k-loops, the stream-K fixups, the epilogues and the start /
end spread of the CTAs.

    python tools/trace_phases.py [--n 1024] [--k K] [--ops NN] [--policy 0] [--beta 1]
"""
import argparse
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_05575_b200 as qg  # noqa: E402
from paper_1903_05575_b200 import _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1024)
ap.add_argument("--k", type=int, default=None)
ap.add_argument("--ops", default="NN")
ap.add_argument("--policy", type=int, default=0)
ap.add_argument("--beta", type=float, default=1.0)
a = ap.parse_args()
lib = _lib.load()
if not hasattr(lib, "qgemm_debug_trace"):
    sys.exit("libqgemm.so was not built with -DQG_TRACE")
lib.qgemm_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
qg.set_path_policy(a.policy)
g = torch.Generator(device="cuda").manual_seed(0)
n, K = a.n, a.k or a.n
ar, ac = (n, K) if a.ops[0] == "N" else (K, n)
br, bc = (K, n) if a.ops[1] == "N" else (n, K)
A = torch.randn((ac, ar, 4), dtype=torch.float64, device="cuda", generator=g)
B = torch.randn((bc, br, 4), dtype=torch.float64, device="cuda", generator=g)
C = torch.randn((n, n, 4), dtype=torch.float64, device="cuda", generator=g)
buf = np.zeros(256 * 48, dtype=np.uint64)
for _ in range(3):
    qg.qgemm(a.ops[0], a.ops[1], 1.0, A, B, a.beta, C, M=n, N=n, K=K)
torch.cuda.synchronize()
lib.qgemm_debug_trace(buf.ctypes.data, buf.size)  # clear
qg.qgemm(a.ops[0], a.ops[1], 1.0, A, B, a.beta, C, M=n, N=n, K=K)
torch.cuda.synchronize()
rc = lib.qgemm_debug_trace(buf.ctypes.data, buf.size)
assert rc == 0, rc
ev = buf.reshape(256, 48)
code = (ev >> np.uint64(56)).astype(int)
t = (ev & np.uint64((1 << 56) - 1)).astype(np.int64)
ctas = [c for c in range(256) if code[c, 0] == 1]
t0 = min(t[c, 0] for c in ctas)
t_end = max(t[c][code[c] == 6].max() for c in ctas)
rows = []
kl_each, epi_each, gap_each, b0_each, b1_each, tail_each, first_each = [], [], [], [], [], [], []  # per traced unit (the first ~46 events of each CTA)
for c in ctas:
    cc, tt = code[c], t[c] - t0
    m = cc > 0
    cc, tt = cc[m], tt[m]
    kloop = fix = epi = 0
    for i in range(len(cc) - 1):
        d = tt[i + 1] - tt[i]
        if cc[i] == 2 and cc[i + 1] == 9:
            first_each.append(int(d))
            k = i + 2
            if k < len(cc) and cc[k] == 3:
                kloop += tt[k] - tt[i]
                kl_each.append(int(tt[k] - tt[i]))
        elif cc[i] == 2 and cc[i + 1] == 3:
            kloop += d
            kl_each.append(int(d))
        elif cc[i] == 3 and cc[i + 1] == 4:
            fix += d
        elif cc[i] == 4 and cc[i + 1] in (5, 7):
            # epilogue start -> (batch 0 data landed | epilogue end)
            j = i + 1
            while j < len(cc) and cc[j] in (7, 8):
                j += 1
            if j < len(cc) and cc[j] == 5:
                epi += tt[j] - tt[i]
                epi_each.append(int(tt[j] - tt[i]))
                if cc[i + 1] == 7 and i + 2 < len(cc) and cc[i + 2] == 8:
                    b0_each.append(int(tt[i + 1] - tt[i]))
                    b1_each.append(int(tt[i + 2] - tt[i + 1]))
                    tail_each.append(int(tt[j] - tt[i + 2]))
        elif cc[i] == 5 and cc[i + 1] == 2:
            gap_each.append(int(d))
    rows.append({"start": int(tt[0]), "end": int(tt[-1]), "kloop": int(kloop), "fixup": int(fix),
                 "epilogue": int(epi), "units": int((cc == 2).sum())})
span = int(t_end - t0)  # (with > 46 events per CTA the sums cover only the traced prefix)
avg = {k: float(np.mean([r[k] for r in rows])) for k in ("start", "kloop", "fixup", "epilogue", "units")}
avg["idle_after_end"] = float(np.mean([span - r["end"] for r in rows]))
print(json.dumps({"n": n, "K": K, "ops": a.ops, "policy": a.policy, "beta": a.beta, "ctas": len(ctas),
                  "span_ns": span, "avg_ns": avg,
                  "frac_of_span": {k: avg[k] / span for k in ("start", "kloop", "fixup", "epilogue", "idle_after_end")},
                  "end_spread_ns": int(max(r["end"] for r in rows) - min(r["end"] for r in rows)),
                  "max_fixup_ns": max(r["fixup"] for r in rows),
                  "epilogue_each_ns_p50_p90": [float(np.percentile(epi_each, 50)), float(np.percentile(epi_each, 90))]
                  if epi_each else None,
                  "kloop_each_ns_p50": float(np.percentile(kl_each, 50)) if kl_each else None,
                  "epilogue_to_next_unit_ns_p50": float(np.percentile(gap_each, 50)) if gap_each else None,
                  "unit_start_to_first_stage_ns_p50_p90": [float(np.percentile(first_each, 50)),
                                                           float(np.percentile(first_each, 90))]
                  if first_each else None,
                  "epi_batch0_wait_p50": float(np.percentile(b0_each, 50)) if b0_each else None,
                  "epi_batch0_work_batch1_wait_p50": float(np.percentile(b1_each, 50)) if b1_each else None,
                  "epi_batch1_work_p50": float(np.percentile(tail_each, 50)) if tail_each else None},
                 indent=1))
