#!/bin/bash
# FP32 A/B: whole-warp MMA issuer with elect.sync (descriptors back in uniform registers)
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x -k "f32 or tc32 or split" > gpurun_out/r2n_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2n_tests.log
SO=paper_1903_05575_b200/libqgemm.so
cp $SO /tmp/cur.so
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  -o /tmp/r01.so _variants/r01csrc/paper_1903_05575_b200/csrc/*.cu _variants/stub_pack_panel.cu
QG_NVCC_EXTRA="-DQG_TC2_CHUNK_KT=100000" python -c "from paper_1903_05575_b200 import build; build.build(force=True)"; cp $SO /tmp/off.so
QG_NVCC_EXTRA="-DQG_TC2_CHUNK_KT=64" python -c "from paper_1903_05575_b200 import build; build.build(force=True)"; cp $SO /tmp/kc64.so
for v in r01 off cur kc64; do
  cp /tmp/$v.so $SO
  python bench.py --no-cpu --no-configs --no-sharded --no-e2e --no-parity --steps 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); v=d['variants']['c3_fp32']
print(json.dumps({'v': '$v', 'c3_fp32_tflops': v['value'], 'ms': v['ms_per_step'], 'clocks': v['clocks']}))" >> gpurun_out/r2n_bench.jsonl
done
cp /tmp/cur.so $SO
python tools/f32_sizes.py > gpurun_out/r2n_sizes.jsonl 2>&1
