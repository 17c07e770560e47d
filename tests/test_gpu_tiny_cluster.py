"""The tile-exact small kernel's cluster-pair variant (qg_small.cuh
qgemm_tiny_kernel<..., 2>: each tile's K split over two CTAs on two SMs, partial
sums through distributed shared memory).  The library reads its switch
(environment variable QG_TINY_Z, else the QG_TINY_CLUSTER build default) once
per process, so the tiny-kernel and c1 parity tests run again in a child
process with QG_TINY_Z=1 (and =0): bitwise against the oracle and against the
general small kernel on exact-integer inputs, every op pair, FP64 and FP32."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("z", ["1", "0"])
def test_tiny_kernel_cluster_pair_parity(z):
    env = dict(os.environ, QG_TINY_Z=z)
    r = subprocess.run([sys.executable, "-m", "pytest", "tests/test_gpu_parity.py", "-m", "gpu", "-q", "-x",
                        "-p", "no:cacheprovider", "-k", "tiny_kernel or c1_full or small_kernel_split"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
    assert " passed" in r.stdout
