"""Sustained tf32 tensor throughput with cuBLAS (torch.matmul, float32 inputs,
TF32 allowed), the way MEASURED_PEAKS.json measures bf16: best of 10 (burst)
and back to back for ~4 s (sustained), with SM clocks / throttle reasons
sampled during the sustained run.  Context measurement for the FP32 (3xTF32)
roofline; not product code.

    python tools/microbench/tf32_cublas.py [--n 8192] [--seconds 4]
"""
import argparse
import json
import statistics
import threading
import time

import torch

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=8192)
ap.add_argument("--seconds", type=float, default=4.0)
a = ap.parse_args()
torch.backends.cuda.matmul.allow_tf32 = True
n = a.n
x = torch.randn(n, n, device="cuda")
y = torch.randn(n, n, device="cuda")
flop = 2.0 * n ** 3
for _ in range(3):
    torch.matmul(x, y)
torch.cuda.synchronize()
best = 0.0
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    torch.matmul(x, y)
    e1.record()
    torch.cuda.synchronize()
    best = max(best, flop / (e0.elapsed_time(e1) * 1e-3) / 1e12)

samples = []
stop = False


def sample():
    import pynvml
    pynvml.nvmlInit()
    h = pynvml.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
    while not stop:
        samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h),
                        pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0))
        time.sleep(0.05)


th = threading.Thread(target=sample)
th.start()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
per = max(1, int(a.seconds / (flop / (best * 1e12))))
e0.record()
for _ in range(per):
    torch.matmul(x, y)
e1.record()
torch.cuda.synchronize()
stop = True
th.join()
sustained = flop * per / (e0.elapsed_time(e1) * 1e-3) / 1e12
clk = [s[0] for s in samples]
print(json.dumps({"tf32_cublas_burst_tflops": best, "tf32_cublas_sustained_tflops": sustained,
                  "n": n, "sustained_calls": per, "sustained_ms": e0.elapsed_time(e1),
                  "sm_mhz_median": statistics.median(clk) if clk else None,
                  "reasons_mask_union": hex(sum({s[1] for s in samples})) if samples else None,
                  "power_w_max": max((s[2] for s in samples), default=None)}))
