#!/bin/bash
# tile-exact small kernel, cluster-pair split (QG_TINY_Z): parity in a child process, A/B latency
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_tiny_cluster.py -m gpu -q > gpurun_out/r2zc_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2zc_tests.log
for r in 1 2; do for z in 0 1; do
  echo "== QG_TINY_Z=$z r$r" >> gpurun_out/r2zc_c1.txt
  QG_TINY_Z=$z timeout 300 python tools/c1_probe.py >> gpurun_out/r2zc_c1.txt 2>&1
done; done
