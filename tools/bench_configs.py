"""Time qgemm on each BASELINE.json config (device-resident inputs, CUDA events).

Context numbers for DESIGN.md / profiles (bench.py times the headline config).
    python tools/bench_configs.py [--configs c1,c2,c3,c4,c5] [--reps 3]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_05575_b200 as qg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="c1,c2,c3,c3f32,c4")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--c5-workspace-gb", type=float, default=16.0)
ap.add_argument("--policy", type=int, default=0, help="qgemm_set_path_policy (0 auto, 1 packed, 2 small, 3 direct)")
a = ap.parse_args()
qg.set_path_policy(a.policy)
dev = torch.device("cuda")
g = torch.Generator(device="cuda").manual_seed(0)


def rnd(cols, ld, dt):
    return (2 * torch.rand((cols, ld, 4), dtype=dt, device=dev, generator=g) - 1)


def timeit(fn, reps):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts), sorted(ts)[len(ts) // 2]


def run(name, M, N, K, opA, opB, alpha, beta, dt=torch.float64, ld=None, ws_cap=None, reps=3):
    ar, ac = (M, K) if opA == "N" else (K, M)
    br, bc = (K, N) if opB == "N" else (N, K)
    A = rnd(ac, ld or ar, dt)
    B = A if name == "c4" else rnd(bc, ld or br, dt)
    C = rnd(N, ld or M, dt)
    fn = qg.qgemm if dt == torch.float64 else qg.qgemm_f32
    need = qg.workspace_bytes(opA, opB, M, N, K, dt)
    if ws_cap and need > ws_cap:
        need = int(ws_cap)
    ws = torch.empty(need, dtype=torch.uint8, device=dev)
    qg.timing_enable(True)
    tmin, tmed = timeit(lambda: fn(opA, opB, alpha, A, B, beta, C, M=M, N=N, K=K, workspace=ws), reps)
    kt = qg.timing_collect()
    qg.timing_enable(False)
    calls = reps + 1
    fl = 32.0 * M * N * K
    out = {"config": name, "M": M, "N": N, "K": K, "ops": opA + opB, "policy": a.policy,
           "dtype": "f64" if dt == torch.float64 else "f32",
           "ms_min": tmin, "ms_med": tmed, "tflops_best": fl / tmin / 1e9,
           "tflops_med": fl / tmed / 1e9,
           "launches_per_call": (kt["pack"][1] + kt["mainloop"][1] + kt["scale"][1]
                                 + kt["small"][1]) // calls,
           "pack_ms_per_call": kt["pack"][0] / calls,
           "main_ms_per_call": (kt["mainloop"][0] + kt["small"][0]) / calls}
    if tmin < 5.0:
        # launch-bound sizes: the same call captured once in a CUDA graph and
        # replayed, so host-side Python/ctypes time is not on the device timeline
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            fn(opA, opB, alpha, A, B, beta, C, M=M, N=N, K=K, workspace=ws)
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=s):
                fn(opA, opB, alpha, A, B, beta, C, M=M, N=N, K=K, workspace=ws)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        nrep = 200
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(nrep):
            gr.replay()
        e1.record()
        torch.cuda.synchronize()
        tg = e0.elapsed_time(e1) / nrep
        out.update({"graph_ms_per_call": tg, "graph_tflops": fl / tg / 1e9})
    print(json.dumps(out), flush=True)
    del A, B, C, ws
    torch.cuda.empty_cache()


for c in a.configs.split(","):
    if c == "c1":
        run("c1", 64, 64, 64, "N", "N", 1.0, 0.0, reps=20)
    elif c == "c2":
        for oa in "NTH":
            for ob in "NTH":
                run("c2", 1024, 1024, 1024, oa, ob, 0.75, -0.5, ld=1040, reps=10)
    elif c == "c3":
        run("c3", 8192, 8192, 8192, "N", "H", 1.0, 1.0, reps=a.reps)
    elif c == "c3f32":
        run("c3", 8192, 8192, 8192, "N", "H", 1.0, 1.0, dt=torch.float32, reps=a.reps)
    elif c == "c4":
        run("c4", 32768, 32768, 256, "N", "H", 1.0, 1.0, reps=a.reps)
    elif c == "c4herk":
        n, K = 32768, 256
        A = rnd(K, n, torch.float64)
        C = rnd(n, n, torch.float64)
        qg.timing_enable(True)
        tmin, tmed = timeit(lambda: qg.qherk("L", "N", 1.0, A, 1.0, C), a.reps)
        kt = qg.timing_collect()
        qg.timing_enable(False)
        fl = 32.0 * n * n * K  # the qgemm-equivalent work, for comparison with c4
        print(json.dumps({"config": "c4herk", "M": n, "N": n, "K": K, "ops": "herk-L-N",
                          "dtype": "f64", "ms_min": tmin, "ms_med": tmed,
                          "tflops_best_gemm_equiv": fl / tmin / 1e9,
                          "tflops_best_actual": fl * (n / 64 + 1) / (2 * n / 64) / tmin / 1e9,
                          "main_ms_per_call": kt["mainloop"][0] / (a.reps + 1)}), flush=True)
        del A, C
        torch.cuda.empty_cache()
    elif c == "c5":
        run("c5", 32768, 32768, 32768, "N", "N", 1.0, 0.0, ws_cap=a.c5_workspace_gb * 1e9, reps=1)
