#!/bin/bash
# FP32 K-panel cap test; c1 with single vs dual accumulators in the tile-exact kernel
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -k "f32_long_k or tiny or c3_full_size_sampled_and_freivalds" > gpurun_out/r2e_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2e_tests.log
python tools/c1_probe.py > gpurun_out/r2e_c1_single.jsonl 2>&1
python tools/f32_accuracy.py > gpurun_out/r2e_f32acc.jsonl 2>&1
QG_NVCC_EXTRA="-DQG_TINY_DUAL=1" python -c "from paper_1903_05575_b200 import build; build.build(force=True)"
python tools/c1_probe.py > gpurun_out/r2e_c1_dual.jsonl 2>&1
