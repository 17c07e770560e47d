"""include/qgemm.h is a plain C header: examples/qgemm_example.c compiles and
links against libqgemm.so with gcc (CPU); it runs and matches on a GPU."""
from __future__ import annotations

import os
import subprocess

import pytest

from paper_1903_05575_b200 import build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def example(tmp_path_factory):
    so = build.build()
    exe = str(tmp_path_factory.mktemp("cex") / "qgemm_example")
    libdir = os.path.dirname(so)
    cmd = ["gcc", "-std=c11", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
           "-I", "/usr/local/cuda/include", os.path.join(ROOT, "examples", "qgemm_example.c"),
           "-L", libdir, "-lqgemm", "-L", "/usr/local/cuda/lib64", "-lcudart", "-lm",
           f"-Wl,-rpath,{libdir}", "-o", exe]
    res = subprocess.run(cmd, capture_output=True, text=True)
    assert res.returncode == 0, res.stderr
    return exe


def test_c_example_builds(example):
    assert os.path.exists(example)


@pytest.mark.gpu
def test_c_example_runs(example):
    res = subprocess.run([example], capture_output=True, text=True, timeout=120)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "OK" in res.stdout
