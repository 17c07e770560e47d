#!/bin/bash
# FP32 chunk fold via L2 reductions (QG_TC2_RED=1) vs slot+fold into C (0): parity + A/B speed
cd $GRAFT_REPO_ROOT
SO=paper_1903_05575_b200/libqgemm.so
cp $SO /tmp/fold.so
QG_NVCC_EXTRA="-DQG_TC2_RED=1" python -c "from paper_1903_05575_b200 import build; build.build(force=True)"; cp $SO /tmp/red.so
timeout 900 python -m pytest tests -m gpu -q -x -k "f32 or tc32 or split" > gpurun_out/r2u_tests_red.log 2>&1
echo "rc=$?" >> gpurun_out/r2u_tests_red.log
F32ACC_N=2048 F32ACC_K=8192 F32ACC_DIST=uniform python tools/f32_accuracy.py > gpurun_out/r2u_acc_red.jsonl 2>&1
for v in fold red fold red; do
  cp /tmp/$v.so $SO
  python bench.py --no-cpu --no-configs --no-sharded --no-e2e --no-parity --steps 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); v=d['variants']['c3_fp32']
print(json.dumps({'v': '$v', 'c3_fp32_tflops': v['value'], 'ms': v['ms_per_step'], 'clocks': v['clocks']}))" >> gpurun_out/r2u_bench.jsonl
done
cp /tmp/red.so $SO; python tools/f32_sizes.py > gpurun_out/r2u_sizes_red.jsonl 2>&1
cp /tmp/fold.so $SO
