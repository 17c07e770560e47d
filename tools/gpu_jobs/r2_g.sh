#!/bin/bash
# FP32 chunk promotion v2 (drain -> slot, fold behind the next chunk): speed vs chunk length, accuracy, tests
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x -k "f32 or tc32 or split" > gpurun_out/r2g_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2g_tests.log
F32ACC_N=2048 python tools/f32_accuracy.py > gpurun_out/r2g_f32acc_2048.jsonl 2>&1
python tools/f32_sizes.py > gpurun_out/r2g_sizes_kc32.txt 2>&1
for kc in 64 128 100000; do
  QG_NVCC_EXTRA="-DQG_TC2_CHUNK_KT=$kc" python -c "from paper_1903_05575_b200 import build; build.build(force=True)"
  python tools/f32_sizes.py > gpurun_out/r2g_sizes_kc$kc.txt 2>&1
done
