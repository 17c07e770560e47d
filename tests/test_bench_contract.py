"""bench.py keeps the driver's JSON-line contract (README "Build, test, benchmark").

The reference arm (the CPU oracle) runs here on CPU; our arm needs a GPU."""
from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True,
                         text=True, timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_json_line():
    line = _run(["--impl", "reference", "--size", "128", "--steps", "1", "--warmup", "1"])
    assert line["impl"] == "reference"
    assert line["unit"] == "TFLOP/s" and line["higher_is_better"] is True and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert line["metric"].startswith("QGEMM FP64 TFLOP/s")


@pytest.mark.gpu
def test_our_arm_json_line():
    line = _run(["--size", "1024", "--steps", "3", "--warmup", "3", "--no-cpu", "--no-sharded"])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "gpu_launches",
                "clocks"):
        assert key in line, key
    assert line["n_gpus"] == 1 and line["steps"] == 3 and line["warmup"] == 3
    assert line["dtype"] == "f64" and line["value"] > 1.0
    assert line["gpu_launches"] >= 3
    r = line["roofline"]
    assert r["bound"] == "tensor" and r["unit"] == "TFLOP/s" and 0 < r["frac"] <= 1.05
    e = line["e2e"]
    assert e["h2d_bytes_per_step"] == 3 * 1024 * 1024 * 32 and e["d2h_bytes_per_step"] == 1024 * 1024 * 32
    assert "workload" in line["config"] and "sm_mhz" in line["clocks"]
    assert line["variants"]["c3_fp32"]["value"] > 1.0
    # the headline workload re-run once from fresh inputs and checked against the oracle
    assert line["parity"]["ok"] is True and line["parity_ok"] is True
    assert line["parity"]["max_err"] <= line["parity"]["tol"]
    assert line["paper_cpu"]["serial_peak_gflops"] == 24.0


def test_reference_arm_and_cpu_baseline_use_one_sampler():
    """the reference arm and cpu_baseline time the same oracle block
    sampler (square blocks of c3's C, full K), so their rates agree."""
    sys.path.insert(0, ROOT)
    import bench
    side = bench.oracle_block_side(256, 0.2)
    assert 128 <= side <= 256 and side % 16 == 0
    dt, fl = bench.oracle_block(256, 128, 128)
    assert fl == 32.0 * 128 * 128 * 256 and dt > 0
