#!/bin/bash
# FP32 chunk running sum by 16-byte vector reductions (red.global.add.v4.f32) vs scalar: parity + A/B
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SO=paper_1903_05575_b200/libqgemm.so
cp _variants/red_v4.so $SO
timeout 1200 python -m pytest tests -m gpu -q -x -k "f32 or tc32 or split or remainder" > gpurun_out/r2x_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2x_tests.log
F32ACC_N=2048 F32ACC_K=8192 F32ACC_DIST=uniform timeout 300 python tools/f32_accuracy.py > gpurun_out/r2x_acc_v4.jsonl 2>&1
for v in red_scalar red_v4 red_scalar red_v4; do
  cp _variants/$v.so $SO
  timeout 600 python bench.py --no-cpu --no-configs --no-sharded --no-e2e --no-parity --steps 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); v=d['variants']['c3_fp32']
print(json.dumps({'v': '$v', 'c3_fp32_tflops': v['value'], 'ms': v['ms_per_step'], 'clocks': v['clocks']}))" >> gpurun_out/r2x_bench.jsonl
done
cp _variants/red_v4.so $SO
timeout 300 python tools/f32_sizes.py > gpurun_out/r2x_f32_sizes_v4.jsonl 2>&1
