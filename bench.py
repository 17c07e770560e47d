#!/usr/bin/env python
"""QGEMM benchmark (BASELINE.json metric: QGEMM FP64 TFLOP/s at 32 flops per
quaternion multiply-add, and % of the B200 FP64 peak, at 1/2/4/8 GPUs).

Headline workload (N=1): BASELINE.json configs[2] ("c3"): M=N=K=8192, opA=N,
opB=H, alpha=beta=1, components i.i.d. N(0,1), FP64 -- the config the north
star's ">=70% of FP64 peak on one GPU at N=8192" target is quoted on.  N GPUs:
weak scaling (R17), rank r owns an 8192-row block of C and A (M =
8192 N), B is broadcast from rank 0 with NCCL every step and each rank's
epilogue stores its row block into rank 0's C over peer memory (dist.py).

A "step" = one qgemm call = the DMMA mainloop fed by TMA straight from the
interleaved storage (rows a2+a3 fused into it) with the fused epilogue (SURVEY
§8(a) rows a1-a5); at N>1 plus the broadcast of B and the collection of C.
Inputs (2.15 GB per matrix) are far larger than the 126 MB L2, so no flush is
needed between steps.  Inputs are drawn on the device by the counter-based
generator (synth/gpu_gen.py; the host twin regenerates any sampled row for the
oracle), so every rank draws only its own shard.

After the timed steps every workload is re-run once (untimed) from freshly
generated inputs and rank 0 checks sampled full rows and a grid of random
entries of C against the oracle (`parity` in the JSON line).

Variants (same JSON line): c3 in FP32 (3xTF32 on tcgen05), c1/c2/c4/QHERK at
their own sizes, the paper's Fig. 4 comparison on B200 (QGEMM(N) vs cuBLAS
ZGEMM(2N)), and at every N the row-block-sharded configs of BASELINE.json:
c4 (strong: the full 32768^2 x 256 update over N GPUs, gather timed apart)
and c5 (weak: M_loc = 4096, N = K = 32768; N = 8 is c5).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "QGEMM FP64 TFLOP/s (32 flops/quat-MAC) and % of FP64 peak at 1/2/4/8 GPU"
# FP64 tensor-pipe peak MEASURED on this pool's B200 with the DMMA.8x8x4 loop of
# tools/microbench/fp64_pipes.cu (profiles/r01_fp64_pipes.txt), clocks at 1965 MHz.
# MEASURED_PEAKS.json has no FP64 entry, so this is the measured denominator;
# the nominal 148 SMs x 64 FMA/clk x 2 x 1.965 GHz = 37.22 is reported beside it.
FP64_DMMA_PEAK_TFLOPS = 37.0
FP64_NOMINAL_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12  # 37.22
# tcgen05.mma kind::tf32 peak MEASURED on this pool's B200 with the MMA loop of
# tools/microbench/tf32_peak.cu (M=128 N=256 K=8, smem-resident operands, ~1.8 s
# back to back: 1117 TFLOP/s; profiles/r01_tf32_peak.txt) -- the nominal 1.1 PF
TF32_PEAK_TFLOPS = 1117.0
# cuBLAS TF32 GEMM (torch.matmul 8192^3, tools/microbench/tf32_cublas.py,
# profiles/r01_tf32_cublas.json): burst 753.6, sustained 614.5 TFLOP/s at a
# 1132 MHz median clock under sw_power_cap -- the library yardstick
TF32_CUBLAS_BURST = 753.6
TF32_CUBLAS_SUSTAINED = 614.5

# The paper's own CPU numbers (context, other hardware; §5).
PAPER_CPU = {
    "hardware": "Intel Xeon E5-2660 (Sandy Bridge) @ 2.20 GHz (max 3.0 GHz), 1 core; "
                "L1/L2/L3 32 kB / 256 kB / 20 MB (P:1572-1576)",
    "serial_peak_gflops": 24.0,
    "hgemm_ref_gflops": 7.0,                          # ~7, memory bound
    "hgemm_optavx_gflops": 21.0,                      # ~21
    "zgemm_mkl_2n_gflops": 22.0,                      # ~22, MKL 18.0u1 serial
    "hgemm_vs_zgemm_2n_time": "HGEMM-OptAVX(N) ~2x faster than ZGEMM-MKL(2N), incl. N > 3000 "
                              "(P:1633-1636, P:1646-1648)",
    "unit": "GFLOP/s at 32 real flops per quaternion multiply-add (DESIGN.md R1)",
    "workload": "square N x N, alpha = 1, beta = 0, FP64 (P:1616-1618)",
}

SEED = 0
VLD = 1 << 32  # virtual leading dimension of the bench's counter-generated matrices:
               # element (i, j) has the same value whatever the (sharded) shape


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--precision", choices=["f64", "f32"], default="f64")
    ap.add_argument("--size", "--n", dest="n", type=int, default=8192,
                    help="M_loc = N = K (default: c3)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--debug-one-device", action="store_true",
                    help="all ranks on cuda:0 with gloo: functional check of the multi-rank "
                         "paths on a 1-GPU box (c4/c5 variants scaled down); its numbers are "
                         "not a measurement")
    ap.add_argument("--collect", choices=["p2p", "nccl"], default="p2p",
                    help="N>1: C row blocks stored into root's C by the epilogue over peer "
                         "memory (p2p, fused) or gathered with NCCL send/recv after compute")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-f32", action="store_true", help="skip the FP32 (tcgen05) variant")
    ap.add_argument("--no-configs", action="store_true", help="skip the c1/c2/c4/Fig. 4 lines")
    ap.add_argument("--no-sharded", action="store_true", help="skip the c4/c5 sharded variants")
    ap.add_argument("--no-parity", action="store_true", help="skip the oracle checks")
    ap.add_argument("--policy", type=int, default=0,
                    help="library path policy for A/B measurements (qgemm_set_path_policy; 0 = auto)")
    return ap.parse_args()


def gen(mid, r0, nrows, c0, ncols, dev, dist, dtype=None):
    """Block of the bench's counter-generated matrix `mid` (synth/gpu_gen.py)."""
    import torch
    from synth.gpu_gen import counter_block
    return counter_block(SEED, mid, VLD, r0, nrows, c0, ncols, dev, dist,
                         dtype=dtype or torch.float64)


def gen_host(mid, rows, cols, dist):
    from synth.inputs import counter_gather_host
    return counter_gather_host(SEED, mid, VLD, rows, cols, dist)


# ------------------------------------------------------------------ clocks
class ClockSampler(threading.Thread):
    """nvidia-smi-equivalent clock/throttle sampling (NVML) during the timed region."""

    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x2: "applications_clocks_setting", 0x10: "sync_boost"}

    def __init__(self, device_index: int, period: float = 0.05):
        super().__init__(daemon=True)
        self.period = period
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self.power = []
        self._halt = threading.Event()
        self.ok = False
        try:
            import pynvml
            import torch
            pynvml.nvmlInit()
            props = torch.cuda.get_device_properties(device_index)
            try:
                bus = f"{props.pci_domain_id:08x}:{props.pci_bus_id:02x}:{props.pci_device_id:02x}.0"
                self.h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
            except Exception:
                self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.nv = pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover - reported in the JSON
            self.err = repr(e)

    def run(self):
        while self.ok and not self._halt.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
                self.power.append(self.nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0)
            except Exception:
                pass
            time.sleep(self.period)

    def stop(self):
        self._halt.set()
        self.join(timeout=2)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "note": getattr(self, "err", "no samples")}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples),
                "power_w_max": round(max(self.power), 1) if self.power else None}


# ------------------------------------------------------------------ oracle timing (CPU)
def oracle_block(n: int, r: int, c: int):
    """The oracle on the r x c top-left block of c3's C (full K = n): rows 0..r of
    op(A) and columns 0..c of op(B) = B^H, drawn on the host by the counter
    generator (synth).  The oracle materialises op(A) (r x K) and op(B) (K x c)
    before its Alg. 1 loops: O((r + c) K) against O(r c K) of arithmetic, < 1%
    for r = c >= 256.  Returns (seconds, flops)."""
    import oracle
    A_s = gen_host(1, np.arange(r), np.arange(n), "normal")          # (K, r, 4): rows of A
    B_s = gen_host(2, np.arange(c), np.arange(n), "normal")          # (K, c, 4): rows of stored B
    C_s = gen_host(3, np.arange(r), np.arange(c), "normal")          # (c, r, 4)
    t0 = time.perf_counter()
    oracle.qgemm("N", "H", r, c, n, (1, 0, 0, 0), A_s, B_s, (1, 0, 0, 0), C_s)
    dt = time.perf_counter() - t0
    return dt, 32.0 * r * c * n


def oracle_block_side(n: int, seconds: float) -> int:
    """Side of a square block of c3 that takes ~`seconds` of oracle time."""
    s = 128
    dt, _ = oracle_block(n, s, s)
    side = int(s * (seconds / max(dt, 1e-3)) ** 0.5)
    return int(max(128, min(n, side // 16 * 16)))


def cpu_baseline(n, seconds):
    import oracle
    side = oracle_block_side(n, seconds)
    dt, fl = oracle_block(n, side, side)
    return {"value": fl / dt / 1e12, "unit": "TFLOP/s", "cores": oracle.max_threads(),
            "kind": "oracle",
            "sample": f"top-left {side} x {side} block of c3's C (full K={n}; {fl:.3e} flops in "
                      f"{dt:.2f} s), oracle/qgemm_oracle.c OpenMP over columns",
            "paper_cpu": PAPER_CPU}


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle
    n = args.n
    per_step = min(20.0, 150.0 / max(1, args.steps + args.warmup))
    side = oracle_block_side(n, per_step)
    for _ in range(args.warmup):
        oracle_block(n, side, side)
    tot_t = tot_f = 0.0
    for _ in range(args.steps):
        t, f = oracle_block(n, side, side)
        tot_t += t
        tot_f += f
    value = tot_f / tot_t / 1e12
    sample = (f"each step: oracle on the top-left {side} x {side} block of c3's C (full K={n}), "
              f"OpenMP on {oracle.max_threads()} host threads (same sampler as cpu_baseline)")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": tot_t / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"c3: QGEMM M=N=K={n} opA=N opB=H alpha=beta=1 N(0,1) (sampled)",
                       "parallelism": "cpu"},
            "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": oracle.max_threads(),
                             "kind": "oracle", "sample": sample, "paper_cpu": PAPER_CPU},
            "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------ rooflines
def _traffic(key, match):
    """ncu DRAM bytes of the captured launch -- only for the workload it was
    captured on (`match`), else None."""
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        return json.load(open(tp)).get(key) if match else None
    except Exception:
        return None


def make_roofline(precision, achieved, main_ms, step_ms, pack_ms, steps, c3_shape=True):
    """Roofline of the dominant kernel.  achieved = algorithmic flops (32 per
    quaternion MAC) per launch / measured mean launch time."""
    if precision == "f64":
        return {"bound": "tensor", "kernel": "qgemm_dmma_kernel", "achieved": achieved,
                "peak": FP64_DMMA_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": (achieved / FP64_DMMA_PEAK_TFLOPS) if achieved else None,
                "traffic": _traffic("f64_mainloop_bytes_per_launch" if pack_ms else
                                    "f64_direct_mainloop_bytes_per_launch", c3_shape),
                "peak_source": "measured DMMA.8x8x4 loop on this pool's B200, "
                               "tools/microbench/fp64_pipes.cu (profiles/r01_fp64_pipes.txt); "
                               "MEASURED_PEAKS.json has no FP64 entry",
                "frac_of_nominal_37_22": (achieved / FP64_NOMINAL_TFLOPS) if achieved else None,
                "kernel_share_of_step": main_ms / step_ms if step_ms else None,
                "pack_ms_per_step": pack_ms / max(1, steps)}
    # FP32: tcgen05 kind::tf32, 3 MMAs per real product (3xTF32)
    mma = 3 * achieved if achieved else None
    return {"bound": "tensor", "kernel": "qgemm_tc32_2cta_kernel", "achieved": mma,
            "peak": TF32_PEAK_TFLOPS, "unit": "TFLOP/s", "frac": (mma / TF32_PEAK_TFLOPS) if mma else None,
            "achieved_algorithmic": achieved,
            "frac_algorithmic": (achieved / TF32_PEAK_TFLOPS) if achieved else None,
            "vs_cublas_tf32": {"burst": TF32_CUBLAS_BURST, "sustained": TF32_CUBLAS_SUSTAINED,
                               "mma_rate_over_sustained": (mma / TF32_CUBLAS_SUSTAINED) if mma else None,
                               "source": "profiles/r01_tf32_cublas.json"},
            "traffic": _traffic("f32_mainloop_bytes_per_launch", c3_shape),
            "peak_source": "measured tcgen05.mma kind::tf32 loop on this pool's B200, "
                           "tools/microbench/tf32_peak.cu (profiles/r01_tf32_peak.txt); achieved "
                           "counts the 3 tf32 MMAs per real product of 3xTF32",
            "kernel_share_of_step": main_ms / step_ms if step_ms else None,
            "pack_ms_per_step": pack_ms / max(1, steps)}


def measure_f32_variant(A, B, C, n, warmup, steps):
    """c3 in FP32 (BASELINE config 3's second precision) on the same inputs,
    rounded to FP32 on the device; device-resident, CUDA events."""
    import torch
    import paper_1903_05575_b200 as qg
    A32, B32, C32 = A.float(), B.float(), C.float()
    ws = qg.get_workspace(qg.workspace_bytes("N", "H", n, n, n, torch.float32), A.device)
    for _ in range(max(1, warmup)):
        qg.qgemm_f32("N", "H", 1.0, A32, B32, 1.0, C32, workspace=ws)
    torch.cuda.synchronize()
    sampler = ClockSampler(A.device.index or 0)
    sampler.start()
    qg.timing_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        qg.qgemm_f32("N", "H", 1.0, A32, B32, 1.0, C32, workspace=ws)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    kt = qg.timing_collect()
    qg.timing_enable(False)
    clocks = sampler.stop()
    fl = 32.0 * n ** 3
    main_ms, main_cnt = kt["mainloop"]
    # per step, not per launch: a step runs the pair kernel and, when the partial
    # last wave splits over K (c3: 50 pairs x 4), its reduce kernel -- both timed
    # as mainloop launches (dividing by the launch count halved the time)
    achieved = fl / (main_ms / max(1, steps) / 1e3) / 1e12 if main_cnt else None
    del A32, B32, C32
    torch.cuda.empty_cache()
    roof = make_roofline("f32", achieved, main_ms, ms, kt["pack"][0], steps, c3_shape=(n == 8192))
    # the MMA-loop peak is at 1965 MHz; under this kernel's power draw the SM
    # clock drops (sw_power_cap), so also report the fraction of the peak at the
    # clock sampled during the timed region
    mhz = (clocks or {}).get("sm_mhz")
    if mhz and roof.get("achieved"):
        roof["peak_at_observed_clock"] = TF32_PEAK_TFLOPS * mhz / 1965.0
        roof["frac_at_observed_clock"] = roof["achieved"] / roof["peak_at_observed_clock"]
    return {"workload": f"c3 FP32: M=N=K={n} opA=N opB=H alpha=beta=1 (inputs = FP64 draws "
                        "rounded to FP32)", "dtype": "f32 (3xTF32 on tcgen05, FP32 accumulate)",
            "value": fl * steps / (ms / 1e3) / 1e12, "unit": "TFLOP/s", "ms_per_step": ms / steps,
            "steps": steps, "launches_per_step": (kt["mainloop"][1] + kt["pack"][1]) / max(1, steps),
            "roofline": roof, "clocks": clocks}


def _timed(fn, reps, warmup=1):
    import torch
    for _ in range(max(1, warmup)):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def _graphed(fn, reps=200, warmup=1):
    import torch
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=s):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    torch.cuda.synchronize()
    return _timed(gr.replay, reps, warmup)


def measure_other_configs(warmup):
    """BASELINE.json configs 1, 2 and 4 at their own sizes (context lines next to
    the c3 headline).  Device-resident inputs, CUDA events; c1 and c2 are also
    replayed from a CUDA graph (host ctypes time off the timeline)."""
    import torch
    import paper_1903_05575_b200 as qg
    dev = torch.device("cuda")
    g = torch.Generator(device="cuda").manual_seed(0)

    def rnd(cols, ld):
        return 2 * torch.rand((cols, ld, 4), dtype=torch.float64, device=dev, generator=g) - 1

    out = {}
    A, B, C = rnd(64, 64), rnd(64, 64), rnd(64, 64)
    qg.qgemm("N", "N", 1.0, A, B, 0.0, C)
    launches = qg.last_launch_count()
    ms = _graphed(lambda: qg.qgemm("N", "N", 1.0, A, B, 0.0, C), warmup=warmup)

    def c1_32():
        for _ in range(32):
            qg.qgemm("N", "N", 1.0, A, B, 0.0, C)
    ms32 = _graphed(c1_32, reps=50, warmup=warmup) / 32
    x = torch.zeros(1, device=dev)
    floor1 = _graphed(lambda: x.add_(1.0), warmup=warmup)

    def triv32():
        for _ in range(32):
            x.add_(1.0)
    floor32 = _graphed(triv32, reps=50, warmup=warmup) / 32
    out["c1"] = {"workload": "c1: 64^3 N/N alpha=1 beta=0", "us_per_call": ms * 1e3,
                 "us_per_call_back_to_back": ms32 * 1e3,
                 "trivial_kernel_us": floor1 * 1e3, "trivial_kernel_back_to_back_us": floor32 * 1e3,
                 "dmma_time_us": 64 * 16 / 1.965e3,  # 64 DMMAs per SM sub-partition at 16 cycles each
                 "note": "latency-bound: 64 output tiles on 64 SMs; floor = a trivial one-element torch "
                         "kernel replayed the same way",
                 "tflops": 32.0 * 64 ** 3 / (ms * 1e-3) / 1e12, "launches_per_call": launches,
                 "timing": "CUDA-graph replay: one call per graph, and 32 calls per graph"}
    n, ld = 1024, 1040
    per_op = {}
    for oa in "NTH":
        for ob in "NTH":
            A, B, C = rnd(n, ld), rnd(n, ld), rnd(n, ld)
            call = (lambda oa=oa, ob=ob, A=A, B=B, C=C:
                    qg.qgemm(oa, ob, 0.75, A, B, -0.5, C, M=n, N=n, K=n))
            ms = _timed(call, 10, warmup)
            per_op[oa + ob] = {"ms": ms, "tflops": 32.0 * n ** 3 / (ms * 1e-3) / 1e12,
                               "graph_ms": _graphed(call, 20, warmup)}
    out["c2"] = {"workload": "c2: 1024^3, all 9 (opA, opB), alpha=0.75 beta=-0.5, ld=1040",
                 "per_op": per_op,
                 "tflops_min": min(v["tflops"] for v in per_op.values()),
                 "tflops_max": max(v["tflops"] for v in per_op.values())}
    del A, B, C
    n, K = 32768, 256
    A = rnd(K, n)
    C = rnd(n, n)
    ms = _timed(lambda: qg.qgemm("N", "H", 1.0, A, A, 1.0, C, M=n, N=n, K=K), 2, warmup)
    ms_herk = _timed(lambda: qg.qherk("L", "N", 1.0, A, 1.0, C), 2, warmup)
    fl = 32.0 * n * n * K
    out["c4"] = {"workload": "c4: M=N=32768 K=256, C <- A A^H + C (B == A)", "qgemm_ms": ms,
                 "qgemm_tflops": fl / (ms * 1e-3) / 1e12, "qherk_lower_ms": ms_herk,
                 "qherk_speedup": ms / ms_herk}
    del A, C
    torch.cuda.empty_cache()
    return out


def measure_fig4(warmup):
    """The paper's Fig. 4 comparison on B200: QGEMM(N) against the
    same product as a complex GEMM on the 2N x 2N embedding (Eq. hc_mat_mult,
    P:598-625), cuBLAS ZGEMM via torch.matmul in complex128; alpha = 1, beta = 0,
    square.  Times do not depend on the values (random operands)."""
    import torch
    import paper_1903_05575_b200 as qg
    out = []
    for n in (1024, 4096):
        A = torch.randn((n, n, 4), dtype=torch.float64, device="cuda")
        B = torch.randn((n, n, 4), dtype=torch.float64, device="cuda")
        C = torch.empty((n, n, 4), dtype=torch.float64, device="cuda")
        q_ms = _timed(lambda: qg.qgemm("N", "N", 1.0, A, B, 0.0, C), 5 if n > 2048 else 20, warmup)
        del A, B, C
        Z1 = torch.randn((2 * n, 2 * n), dtype=torch.complex128, device="cuda")
        Z2 = torch.randn((2 * n, 2 * n), dtype=torch.complex128, device="cuda")
        Z3 = torch.empty_like(Z1)
        z_ms = _timed(lambda: torch.matmul(Z1, Z2, out=Z3), 5 if n > 2048 else 20, warmup)
        del Z1, Z2, Z3
        torch.cuda.empty_cache()
        fl = 32.0 * n ** 3
        out.append({"N": n, "qgemm_ms": q_ms, "zgemm_2n_ms": z_ms,
                    "qgemm_tflops": fl / (q_ms * 1e-3) / 1e12,
                    "zgemm_2n_tflops_real": 8.0 * (2 * n) ** 3 / (z_ms * 1e-3) / 1e12,
                    "time_ratio_zgemm_over_qgemm": z_ms / q_ms})
    return {"what": "QGEMM(N) vs cuBLAS ZGEMM(2N) on the complex embedding (paper Fig. 4, "
                    "P:1611-1649; the paper reports ~2x on Sandy Bridge with MKL)",
            "points": out}


# ------------------------------------------------------------------ parity (oracle)
def _tol_f64(K, maxa, maxb, maxc0, beta_norm):
    """North-star FP64 tolerance (+ reading R8's beta C0 term)."""
    return 1e-12 * K * maxa * maxb + (8 * 2.0 ** -53 * beta_norm * maxc0 * 4 if beta_norm else 0.0)


def parity_rows_grid(C_cols_rows, M, N, K, rows, grid_rows, grid_cols, a_rows_host, b_cols_panels,
                     b_cols_host, c0_host, transB, beta, rows_what):
    """Compare full rows `rows` and a grid of entries of the device result
    against the oracle.

    C_cols_rows(cols_idx, rows_idx) -> numpy (len(cols), len(rows), 4) of the result;
    a_rows_host(rows) -> stored rows of A (K, len, 4) (op N);
    b_cols_panels() -> iterator over (j0, stored B panel) covering all N columns
      (stored B is N x K for op H: panel (K, nj, 4); K x N for op N: (nj, K, 4));
    b_cols_host(cols) -> the same for selected columns; c0_host(rows, cols) -> C0
    entries (len(cols), len(rows), 4) or None (beta = 0)."""
    import oracle
    A_S = a_rows_host(rows)
    C0_S = c0_host(rows, np.arange(N)) if beta else None
    got_S = C_cols_rows(np.arange(N), rows)
    err, maxb = 0.0, 0.0
    for j0, Bp in b_cols_panels():
        nj = Bp.shape[1] if transB == "H" else Bp.shape[0]
        ref = (np.ascontiguousarray(C0_S[j0:j0 + nj]) if beta else np.zeros((nj, rows.size, 4)))
        oracle.qgemm("N", transB, rows.size, nj, K, 1, A_S, np.ascontiguousarray(Bp), beta, ref)
        err = max(err, float(np.abs(got_S[j0:j0 + nj] - ref).max()))
        maxb = max(maxb, float(np.abs(Bp).max()))
    A_G = a_rows_host(grid_rows)
    B_G = b_cols_host(grid_cols)
    ref = c0_host(grid_rows, grid_cols).copy() if beta else np.zeros((grid_cols.size, grid_rows.size, 4))
    maxc0 = max(float(np.abs(C0_S).max()), float(np.abs(ref).max())) if beta else 0.0
    oracle.qgemm("N", transB, grid_rows.size, grid_cols.size, K, 1, A_G, B_G, beta, ref)
    err = max(err, float(np.abs(C_cols_rows(grid_cols, grid_rows) - ref).max()))
    maxa = max(float(np.abs(A_S).max()), float(np.abs(A_G).max()))
    # max|A| over the sampled rows <= the global max: a stricter tolerance
    tol = _tol_f64(K, maxa, maxb, maxc0, abs(beta))
    return {"ok": bool(err <= tol), "max_err": err, "tol": tol,
            "checked": f"{rows_what} ({rows.size} full rows of {N} entries) + a "
                       f"{grid_rows.size}x{grid_cols.size} grid of random entries vs the oracle "
                       "(oracle/, inputs regenerated by synth's counter generator)"}


def pick(Cdev, cols, rows):
    """Entries (rows x cols) of a device result stored (N, ld, 4), to the host
    as (len(cols), len(rows), 4) -- rows first, so no full copy is made."""
    import torch
    r = torch.from_numpy(np.asarray(rows, dtype=np.int64)).to(Cdev.device)
    c = torch.from_numpy(np.asarray(cols, dtype=np.int64)).to(Cdev.device)
    return Cdev.index_select(1, r).index_select(0, c).cpu().numpy()


def rank_rows(M, world, per_rank_mid=True):
    """First, middle and last row of every rank's block (dist.rows_for_rank)."""
    from paper_1903_05575_b200.dist import rows_for_rank
    out = []
    for r in range(world):
        r0, r1 = rows_for_rank(M, world, r)
        if r1 > r0:
            out += [r0, r1 - 1] + ([r0 + (r1 - r0) // 2 + 1] if per_rank_mid and r1 - r0 > 2 else [])
    return np.unique(np.asarray(out, dtype=np.int64))


def _b_panels_dev(mid, N, K, dist, opB, dev, panel=1024):
    """Stored B regenerated on the device panel by panel and copied to the host
    (fresh tensors from the same generator; synth/gpu_gen.py)."""
    def it():
        for j0 in range(0, N, panel):
            nj = min(panel, N - j0)
            if opB == "H":       # stored N x K: rows j0.. of B, all k -> (K, nj, 4)
                yield j0, gen(mid, j0, nj, 0, K, dev, dist).cpu().numpy()
            else:                # stored K x N: columns j0.. -> (nj, K, 4)
                yield j0, gen(mid, 0, K, j0, nj, dev, dist).cpu().numpy()
    return it


# ------------------------------------------------------------------ multi-rank plumbing
class Ctx:
    def __init__(self, args):
        import torch
        import torch.distributed as dist
        self.args = args
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        local = int(os.environ.get("LOCAL_RANK", "0"))
        if args.debug_one_device:
            local = 0  # functional check of the N>1 code paths on a 1-GPU box (no timing claim)
        self.local = local
        torch.cuda.set_device(local)
        self.dev = torch.device("cuda", local)
        if self.world > 1:
            if args.debug_one_device:
                dist.init_process_group("gloo")
            else:
                dist.init_process_group("nccl", device_id=self.dev)
        self.dist = dist

    def barrier(self):
        import torch
        if self.world > 1:
            if self.args.debug_one_device:
                self.dist.barrier()
            else:
                self.dist.barrier(device_ids=[self.local])
        torch.cuda.synchronize(self.dev)

    def max_over_ranks(self, v):
        import torch
        if self.world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=self.dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def all_ok(self, ok: bool) -> bool:
        import torch
        if self.world == 1:
            return ok
        t = torch.tensor([1 if ok else 0], dtype=torch.int32, device=self.dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN)
        return bool(t.item())

    def peer(self, C_full):
        """Root's C mapped into every rank (dist.PeerC), or None on every rank if
        any rank cannot map it (no P2P / IPC between these GPUs)."""
        from paper_1903_05575_b200.dist import PeerC
        ok, peer = True, None
        try:
            peer = PeerC(C_full)
        except Exception as exc:  # noqa: BLE001 -- reported, then the collective decision below
            print(f"[rank {self.rank}] peer mapping of root's C failed ({exc}); using the NCCL gather",
                  file=sys.stderr)
            ok = False
        if not self.all_ok(ok):
            if peer is not None:
                peer.close()
            return None
        return peer

    def close_peer(self, peer):
        if peer is not None:  # root's C must outlive the peers' mappings
            self.dist.barrier()
            peer.close()
            self.dist.barrier()


def timed_steps(ctx, step, warmup, steps, sample_clocks=False):
    """W untimed steps, then K steps bracketed by barrier + synchronize, CUDA
    events on the launching stream, max over ranks."""
    import torch
    import paper_1903_05575_b200 as qg
    stream = torch.cuda.current_stream(ctx.dev)
    for _ in range(warmup):
        step()
    ctx.barrier()
    sampler = ClockSampler(ctx.local) if sample_clocks else None
    if sampler:
        sampler.start()
    qg.timing_enable(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches = 0
    ctx.barrier()
    e0.record(stream)
    for _ in range(steps):
        launches += step() or 0
    e1.record(stream)
    ctx.barrier()
    ms = ctx.max_over_ranks(e0.elapsed_time(e1))
    kt = qg.timing_collect()
    qg.timing_enable(False)
    clocks = sampler.stop() if sampler else None
    return ms, kt, launches, clocks


# ------------------------------------------------------------------ c5 weak / c4 sharded
def measure_c5_weak(ctx, m_loc, n, warmup, steps, check):
    """BASELINE c5 sharded as SURVEY §8(e)'s weak series: rank r owns M_loc rows,
    N = K = n (32768); G = 8 with M_loc = 4096 is c5 itself.  Per step: NCCL
    broadcast of B (34 GB) + local QGEMM (alpha = 1, beta = 0) whose epilogue
    stores into root's NaN-filled C over peer memory (or the NCCL gather)."""
    import torch
    import paper_1903_05575_b200 as qg
    from paper_1903_05575_b200.dist import qgemm_rowsharded, qgemm_rowsharded_p2p, rows_for_rank
    world, rank, dev = ctx.world, ctx.rank, ctx.dev
    M = m_loc * world
    r0, r1 = rows_for_rank(M, world, rank)
    A_r = gen(11, r0, r1 - r0, 0, n, dev, "uniform")                    # rows of A: (K, m, 4)
    B = gen(12, 0, n, 0, n, dev, "uniform") if rank == 0 else torch.empty((n, n, 4), dtype=torch.float64,
                                                                          device=dev)
    C_full = torch.full((n, M, 4), float("nan"), dtype=torch.float64, device=dev) if rank == 0 else None
    peer = ctx.peer(C_full) if world > 1 and ctx.args.collect == "p2p" else None
    C_r = None
    if world == 1:
        C_r = C_full
    elif peer is None:
        C_r = torch.full((n, r1 - r0, 4), float("nan"), dtype=torch.float64, device=dev)
    ws = qg.get_workspace(qg.workspace_bytes("N", "N", r1 - r0, n, n), dev)

    def step():
        if world == 1:
            qg.qgemm("N", "N", 1.0, A_r, B, 0.0, C_r, workspace=ws)
        elif peer is not None:
            qgemm_rowsharded_p2p("N", "N", 1.0, A_r, B, 0.0, peer, M, n, n, workspace=ws)
        else:
            qgemm_rowsharded("N", "N", 1.0, A_r, B, 0.0, C_r, M, n, n, C_full=C_full,
                             local_gemm=lambda *a, **k: qg.qgemm(*a, workspace=ws, **k))
        return qg.last_launch_count()

    ms, kt, launches, _ = timed_steps(ctx, step, warmup, steps)
    main_ms, main_cnt = kt["mainloop"]
    fl = 32.0 * M * n * n
    res = {"workload": f"c5 weak (SURVEY §8(e)): M = {world} x {m_loc}, N = K = {n}, N/N, alpha=1 "
                       "beta=0 (C NaN-filled), U[-1,1] counter draws",
           "value": fl * steps / (ms / 1e3) / 1e12, "unit": "TFLOP/s", "ms_per_step": ms / steps,
           "steps": steps, "n_gpus": world,
           "per_gpu_tflops": fl / world * steps / (ms / 1e3) / 1e12,
           "mainloop_ms_per_step_rank0": main_ms / max(1, steps),
           "timed": ("NCCL broadcast(B) + local qgemm" + (
               " with epilogue stores into root's C over peer memory + completion all_reduce"
               if peer is not None else " + NCCL gather of C")) if world > 1 else "qgemm",
           "launches_per_step": launches / max(1, steps)}
    del B
    torch.cuda.empty_cache()
    if check and rank == 0:
        K = n
        res["parity"] = parity_rows_grid(
            lambda cols, rows: pick(C_full, cols, rows),
            M, n, K, rank_rows(M, world), np.sort(np.random.default_rng(1).choice(M, 64, replace=False)),
            np.sort(np.random.default_rng(2).choice(n, 64, replace=False)),
            lambda rows: gen_host(11, rows, np.arange(K), "uniform"),
            _b_panels_dev(12, n, K, "uniform", "N", dev),
            lambda cols: gen_host(12, np.arange(K), cols, "uniform"),
            None, "N", 0.0, "first, middle and last row of every rank's block")
        res["parity"]["finite"] = bool(torch.isfinite(C_full).all())    # beta = 0: C never read
        res["parity"]["ok"] = res["parity"]["ok"] and res["parity"]["finite"]
    ctx.close_peer(peer)
    del A_r, C_full, C_r
    torch.cuda.empty_cache()
    return res


def measure_c4_sharded(ctx, n, K, warmup, steps, check):
    """BASELINE c4 row-block sharded (strong): C <- A A^H + C, M = N = n, K, B == A
    broadcast from root; rank r's op(A) rows are a strided VIEW of the broadcast A
    (lda = n); C_r (the rank's rows of the Hermitian C) stays local
    and the gather of the 34 GB result to root is timed separately (§8(e): a
    distributed Hamiltonian build would leave it sharded)."""
    import torch
    import paper_1903_05575_b200 as qg
    from paper_1903_05575_b200.dist import qgemm_rowsharded, rows_for_rank
    from synth.gpu_gen import counter_hermitian
    world, rank, dev = ctx.world, ctx.rank, ctx.dev
    r0, r1 = rows_for_rank(n, world, rank)
    A = gen(21, 0, n, 0, K, dev, "uniform") if rank == 0 else torch.empty((K, n, 4), dtype=torch.float64,
                                                                          device=dev)

    def fresh_c():
        return counter_hermitian(SEED, 23, n, dev, r0=r0, nrows=r1 - r0)

    C_r = fresh_c()
    A_r = A[:, r0:r1, :]
    ws = qg.get_workspace(qg.workspace_bytes("N", "H", r1 - r0, n, K), dev)

    def step():
        if world == 1:
            qg.qgemm("N", "H", 1.0, A_r, A, 1.0, C_r, M=n, N=n, K=K, workspace=ws)
        else:
            qgemm_rowsharded("N", "H", 1.0, A_r, A, 1.0, C_r, n, n, K, gather=False,
                             local_gemm=lambda *a, **k: qg.qgemm(*a, workspace=ws, **k))
        return qg.last_launch_count()

    ms, kt, launches, _ = timed_steps(ctx, step, warmup, steps)
    fl = 32.0 * n * n * K
    res = {"workload": f"c4 strong: M = N = {n}, K = {K}, C <- A A^H + C (B == A broadcast, "
                       f"A_r a strided view, lda = {n}), C Hermitian-initialised, over {world} GPU(s)",
           "value": fl * steps / (ms / 1e3) / 1e12, "unit": "TFLOP/s", "ms_per_step": ms / steps,
           "steps": steps, "n_gpus": world,
           "timed": "NCCL broadcast(A) + local qgemm per step (gather timed separately)"
                    if world > 1 else "qgemm",
           "launches_per_step": launches / max(1, steps)}
    # collection: gather of every row block into root's column-major C (once, timed)
    C_full = None
    if world > 1:
        C_full = torch.empty((n, n, 4), dtype=torch.float64, device=dev) if rank == 0 else None
        C_r.copy_(fresh_c())                                  # verification run from fresh C0
        ctx.barrier()
        step()
        ctx.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        qgemm_rowsharded("N", "H", 1.0, A_r, A, 1.0, C_r, n, n, K, broadcast_b=False, gather=True,
                         C_full=C_full, local_gemm=lambda *a, **k: None)
        e1.record()
        ctx.barrier()
        g_ms = ctx.max_over_ranks(e0.elapsed_time(e1))
        res["gather_ms"] = g_ms
        res["gather_GBps_into_root"] = 32.0 * n * (n - (r1 - r0)) / (g_ms * 1e-3) / 1e9 \
            if rank == 0 else None
        res["value_incl_gather"] = fl / ((ms / steps + g_ms) * 1e-3) / 1e12
    else:
        C_r.copy_(fresh_c())
        step()
        torch.cuda.synchronize()
        C_full = C_r
    if check and rank == 0:
        from synth.inputs import counter_gather_host

        def c0_host(rows, cols):
            i = np.asarray(rows, dtype=np.int64)
            j = np.asarray(cols, dtype=np.int64)
            xij = counter_gather_host(SEED, 23, n, i, j)                         # X_ij
            xji = counter_gather_host(SEED, 23, n, j, i).transpose(1, 0, 2)     # X_ji at [j, i]
            return 0.5 * (xij + np.array([1.0, -1.0, -1.0, -1.0]) * xji)

        A_h = gen_host(21, np.arange(n), np.arange(K), "uniform")             # (K, n, 4), 268 MB
        res["parity"] = parity_rows_grid(
            lambda cols, rows: pick(C_full, cols, rows),
            n, n, K, rank_rows(n, world), np.sort(np.random.default_rng(3).choice(n, 64, replace=False)),
            np.sort(np.random.default_rng(4).choice(n, 64, replace=False)),
            lambda rows: np.ascontiguousarray(A_h[:, rows, :]),
            lambda: iter([(j0, np.ascontiguousarray(A_h[:, j0:j0 + 4096, :])) for j0 in range(0, n, 4096)]),
            lambda cols: np.ascontiguousarray(A_h[:, cols, :]),
            c0_host, "H", 1.0, "first, middle and last row of every rank's block")
    del A, C_r, C_full
    torch.cuda.empty_cache()
    return res


# ------------------------------------------------------------------ our arm
def run_ours(args):
    import torch

    import paper_1903_05575_b200 as qg
    from paper_1903_05575_b200.dist import qgemm_rowsharded, qgemm_rowsharded_p2p, rows_for_rank

    ctx = Ctx(args)
    world, rank, dev = ctx.world, ctx.rank, ctx.dev
    if args.policy:
        qg.set_path_policy(args.policy)
    n = args.n
    M_total = n * world
    r0, r1 = rows_for_rank(M_total, world, rank) if world > 1 else (0, n)
    assert r1 - r0 == n  # n is a multiple of the 64-row tile: every rank owns exactly n rows
    dt = torch.float64 if args.precision == "f64" else torch.float32
    fn = qg.qgemm if args.precision == "f64" else qg.qgemm_f32

    # inputs on the device (counter generator, N(0,1)): A rows r0.., B (root), C
    A = gen(1, r0, n, 0, n, dev, "normal", dt)                     # stored rows of A: (K, n, 4)
    B = gen(2, 0, n, 0, n, dev, "normal", dt) if rank == 0 else torch.empty((n, n, 4), dtype=dt,
                                                                           device=dev)
    C = gen(3, r0, n, 0, n, dev, "normal", dt)
    C_full = torch.empty((n, M_total, 4), dtype=dt, device=dev) if (world > 1 and rank == 0) else None

    def reset_c():
        """C <- C0 (beta = 1 accumulates: the verification run starts fresh)."""
        if C_full is not None:
            C_full.copy_(gen(3, 0, M_total, 0, n, dev, "normal", dt))
        C.copy_(gen(3, r0, n, 0, n, dev, "normal", dt))

    peer = None
    if world > 1 and args.collect == "p2p":
        # C lives on root: each rank's epilogue stores into it over peer memory
        if rank == 0:
            reset_c()
        peer = ctx.peer(C_full)
    ws = qg.get_workspace(qg.workspace_bytes("N", "H", n, n, n, dt), dev)

    def step():
        if world == 1:
            fn("N", "H", 1.0, A, B, 1.0, C, workspace=ws)
            return qg.last_launch_count()
        if peer is not None:
            qgemm_rowsharded_p2p("N", "H", 1.0, A, B, 1.0, peer, M_total, n, n, workspace=ws)
            return qg.last_launch_count()
        qgemm_rowsharded("N", "H", 1.0, A, B, 1.0, C, M_total, n, n, C_full=C_full,
                         local_gemm=lambda *a, **k: fn(*a, workspace=ws, **k))
        return qg.last_launch_count()

    ms, kt, launches, clocks = timed_steps(ctx, step, args.warmup, args.steps, sample_clocks=True)
    flops_step = 32.0 * M_total * n * n
    value = flops_step * args.steps / (ms / 1e3) / 1e12
    main_ms, main_cnt = kt["mainloop"]
    pack_ms, pack_cnt = kt["pack"]
    # the mainloop launches of one step (FP64 c3: one DMMA launch; FP32: the
    # pair kernel + its split-K reduce) against one rank's flops per step
    main_avg_s = main_ms / max(1, args.steps) / 1e3
    achieved = 32.0 * n * n * n / main_avg_s / 1e12 if main_cnt else None
    roofline = make_roofline(args.precision, achieved, main_ms, ms, pack_ms, args.steps,
                             c3_shape=(n == 8192))

    # ---------------- oracle check of the headline workload (one fresh, untimed step)
    parity = None
    if not args.no_parity and args.precision == "f64":
        reset_c()
        ctx.barrier()
        step()
        ctx.barrier()
        if rank == 0:
            Cres = C_full if C_full is not None else C
            parity = parity_rows_grid(
                lambda cols, rows: pick(Cres, cols, rows),
                M_total, n, n, rank_rows(M_total, world),
                np.sort(np.random.default_rng(5).choice(M_total, 64, replace=False)),
                np.sort(np.random.default_rng(6).choice(n, 64, replace=False)),
                lambda rows: gen_host(1, rows, np.arange(n), "normal"),
                _b_panels_dev(2, n, n, "normal", "H", dev, panel=n),
                lambda cols: gen_host(2, cols, np.arange(n), "normal"),
                lambda rows, cols: gen_host(3, rows, cols, "normal"), "H", 1.0,
                "first, middle and last row of every rank's block")
            parity["inputs"] = ("counter-based N(0,1) draws (synth: Box-Muller on splitmix64); the "
                                "oracle's rows of A / C0 from the numpy twin, B regenerated on the "
                                "device by the torch twin (equal to a few ulp)")
        ctx.barrier()

    # ---------------- e2e through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        pinA = A.cpu().pin_memory()
        pinB = B.cpu().pin_memory()
        pinC = C.cpu().pin_memory()
        outC = (torch.empty(C_full.shape if C_full is not None else C.shape, dtype=dt).pin_memory()
                if world > 1 else None)
        e_steps = max(1, min(args.steps, 3))
        stream = torch.cuda.current_stream(dev)

        host_ws = None
        if world == 1:
            host_ws = torch.empty(qg.host_workspace_bytes("N", "H", n, n, n, dt), dtype=torch.uint8,
                                  device=dev)

        def e2e_step():
            if world == 1:
                # the library's end-to-end call: host A/B/C streamed through device
                # staging, transfers overlapped with the mainloop (qgemm_host)
                qg.qgemm_host("N", "H", 1.0, pinA, pinB, 1.0, pinC, workspace=host_ws)
                return
            A.copy_(pinA, non_blocking=True)
            if rank == 0:
                B.copy_(pinB, non_blocking=True)
            if peer is None:
                C.copy_(pinC, non_blocking=True)
            elif rank == 0:
                for r in range(world):  # C lives on root: upload every row block
                    C_full[:, r * n:(r + 1) * n, :].copy_(pinC, non_blocking=True)
            step()
            src = C_full if C_full is not None else C
            if rank == 0:
                outC.copy_(src, non_blocking=True)

        e2e_step()
        ctx.barrier()
        f0 = torch.cuda.Event(enable_timing=True)
        f1 = torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(e_steps):
            e2e_step()
        f1.record(stream)
        ctx.barrier()
        ems = ctx.max_over_ranks(f0.elapsed_time(f1))
        el = A.element_size()
        h2d = (A.numel() + C.numel()) * el * world + B.numel() * el  # same bytes either way
        d2h = (C_full.numel() if C_full is not None else C.numel()) * el
        e2e = {"value": flops_step * e_steps / (ems / 1e3) / 1e12, "unit": "TFLOP/s",
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "steps": e_steps, "ms_per_step": ems / e_steps,
               "path": ("pinned host -> qgemm_host C ABI (K-chunked H2D / column-panel D2H "
                        "overlapped with the mainloop) -> pinned host") if world == 1 else
                       f"pinned host -> qgemm_rowsharded{'_p2p' if peer is not None else ''} -> "
                       "pinned host"}
        del pinA, pinB, pinC, outC, host_ws

    variants = {}
    if world == 1 and args.precision == "f64" and not args.no_f32:
        variants["c3_fp32"] = measure_f32_variant(A, B, C, n, args.warmup, args.steps)
    ctx.close_peer(peer)
    del A, B, C, C_full, ws
    torch.cuda.empty_cache()
    if world == 1 and args.precision == "f64" and not args.no_configs and n == 8192:
        variants["other_configs"] = measure_other_configs(args.warmup)
        variants["fig4_b200"] = measure_fig4(args.warmup)
    if args.precision == "f64" and not args.no_sharded:
        small = args.debug_one_device
        check = not args.no_parity
        variants["c4_sharded"] = measure_c4_sharded(ctx, 4096 if small else 32768, 256, 1, 2, check)
        variants["c5_weak"] = measure_c5_weak(ctx, 1024 if small else 4096, 4096 if small else 32768,
                                              1, 2, check)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(n, args.cpu_seconds)

    if rank == 0:
        oks = [p["parity"]["ok"] for p in variants.values() if isinstance(p, dict) and "parity" in p]
        if parity is not None:
            oks.append(parity["ok"])
        line = {"metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": args.precision, "data": "synthetic",
                "pct_of_fp64_peak": 100.0 * value / (FP64_DMMA_PEAK_TFLOPS * world)
                if args.precision == "f64" else None,
                "pct_of_fp64_nominal": 100.0 * value / (FP64_NOMINAL_TFLOPS * world)
                if args.precision == "f64" else None,
                "config": {"workload": f"c3: QGEMM M={M_total} (={world}x{n}) N=K={n} opA=N opB=H "
                                       "alpha=beta=1 N(0,1) components, column-major interleaved",
                           "global_batch": 1, "seq_len": None,
                           "parallelism": f"rowblock{world}" + (
                               ("+bcastB+p2p-epilogue-into-root-C" if peer is not None
                                else "+bcastB+gatherC") if world > 1 else ""),
                           "l2": "inputs (2.15 GB/matrix) >> 126 MB L2; no flush",
                           "timed": ("pack A + pack B + DMMA mainloop/epilogue per step" if pack_cnt else
                                     "TMA-fed DMMA mainloop/epilogue (no pack) per step")
                                    + ((" + NCCL broadcast(B) + epilogue stores into root's C "
                                        "over NVLink + completion all_reduce" if peer is not None
                                        else " + NCCL broadcast(B) + gather(C)")
                                       if world > 1 else "")},
                "parity": parity, "parity_ok": bool(oks) and all(oks) if oks else None,
                "roofline": roofline, "cpu_baseline": cpu, "paper_cpu": PAPER_CPU, "e2e": e2e,
                "variants": variants, "gpu_launches": launches, "clocks": clocks,
                "library": qg.version()}
        print(json.dumps(line), flush=True)
    if world > 1:
        ctx.dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
