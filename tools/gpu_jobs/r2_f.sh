#!/bin/bash
# FP32 pair kernel with accumulation chunks: parity (all FP32 tests), accuracy vs K, speed
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q -x -k "f32 or tc32 or split or host" > gpurun_out/r2f_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2f_tests.log
python tools/f32_accuracy.py > gpurun_out/r2f_f32acc.jsonl 2>&1
F32ACC_N=2048 python tools/f32_accuracy.py > gpurun_out/r2f_f32acc_2048.jsonl 2>&1
python tools/f32_sizes.py > gpurun_out/r2f_f32_sizes.txt 2>&1
python bench.py --no-cpu --no-configs --no-sharded --no-e2e --steps 5 > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err
