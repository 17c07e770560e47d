"""Build libqgemm.so in-tree with nvcc for sm_100a (no JIT cache, no torch ext).

    python -m paper_1903_05575_b200.build
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
SO = os.path.join(PKG, "libqgemm.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [
        os.path.join(os.path.dirname(PKG), "include", "qgemm.h")]


def needs_build() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(d) > t for d in deps())


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return SO
    tmp = SO + f".tmp{os.getpid()}"
    extra = os.environ.get("QG_NVCC_EXTRA", "").split()  # tuning experiments only
    cmd = [NVCC, *ARCH, *FLAGS, *extra, "-o", tmp, *sources()]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libqgemm.so")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(tmp, SO)
    return SO


def build_variant(out: str, extra_flags: list[str]) -> str:
    """Build the same sources with extra nvcc flags into `out` (tests only:
    e.g. the negative-control library, -DQG_NEGATIVE_CONTROL)."""
    cmd = [NVCC, *ARCH, *FLAGS, *extra_flags, "-o", out, *sources()]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed building {out}")
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
