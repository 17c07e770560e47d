"""FP32 path accuracy vs K: error of qgemm_f32 (3xTF32 on tcgen05) against the
FP64 oracle on the FP64 inputs (reading R11), as a fraction of the north-star
FP32 tolerance and against the error of the same inputs rounded to FP32 and
multiplied exactly (the input-rounding floor).  N(0,1) inputs, N/H, beta = 0.

    python tools/f32_accuracy.py
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (test infrastructure: this tool measures, it is not product code)
import paper_1903_05575_b200 as qg  # noqa: E402
from synth import make_problem  # noqa: E402


def main():
    n = int(os.environ.get("F32ACC_N", "512"))
    dist = os.environ.get("F32ACC_DIST", "normal")     # normal | uniform | int2 (entries in {-2..2})
    Ks = [int(k) for k in os.environ.get("F32ACC_K", "64,256,1024,4096,8192").split(",")]
    for K in Ks:
        pr = make_problem(n, n, K, "N", "H", 1, 0, seed=1, dist=dist)
        A = torch.from_numpy(pr.A).cuda().float()
        B = torch.from_numpy(pr.B).cuda().float()
        C = torch.zeros((n, n, 4), dtype=torch.float32, device="cuda")
        qg.qgemm_f32("N", "H", 1.0, A, B, 0.0, C)
        got = C.double().cpu().numpy()
        ref = np.zeros((n, n, 4))
        oracle.qgemm("N", "H", n, n, K, 1, pr.A, pr.B, 0, ref)
        ref32 = np.zeros((n, n, 4))   # exact product of the FP32-rounded inputs
        oracle.qgemm("N", "H", n, n, K, 1, A.double().cpu().numpy(), B.double().cpu().numpy(), 0, ref32)
        e = got - ref
        tol = 1e-4 * K ** 0.5 * np.abs(pr.A).max() * np.abs(pr.B).max()
        print(json.dumps({"K": K, "M=N": n, "dist": dist, "max_err": float(np.abs(e).max()), "std_err": float(e.std()),
                          "mean_err": float(e.mean()), "tol": tol, "max_over_tol": float(np.abs(e).max() / tol),
                          "input_rounding_max_err": float(np.abs(ref32 - ref).max()),
                          "kernel_max_err_vs_rounded_inputs": float(np.abs(got - ref32).max()),
                          "rms_C": float(np.sqrt((ref ** 2).mean()))}), flush=True)


if __name__ == "__main__":
    main()
