#!/bin/bash
# FP32 accuracy vs accumulation chunk (k-tiles) and input distribution, M = N = 2048, K = 8192
cd $GRAFT_REPO_ROOT
for kc in 32 64 128 100000; do
  QG_NVCC_EXTRA="-DQG_TC2_CHUNK_KT=$kc" python -c "from paper_1903_05575_b200 import build; build.build(force=True)"
  for d in normal uniform int2; do
    F32ACC_N=2048 F32ACC_K=8192 F32ACC_DIST=$d python tools/f32_accuracy.py | sed "s/^{/{\"kc\": $kc, /" >> gpurun_out/r2h_acc.jsonl 2>&1
  done
  python tools/f32_sizes.py | sed "s/^{/{\"kc\": $kc, /" >> gpurun_out/r2h_sizes.jsonl 2>&1
done
