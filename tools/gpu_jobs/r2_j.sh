#!/bin/bash
# FP32 A/B on one box: round-1 library (no chunks) vs the current one (kc 32, 64)
cd $GRAFT_REPO_ROOT
SO=paper_1903_05575_b200/libqgemm.so
cp $SO /tmp/cur.so
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
  -o /tmp/r01.so _variants/r01csrc/paper_1903_05575_b200/csrc/*.cu
QG_NVCC_EXTRA="-DQG_TC2_CHUNK_KT=64" python -c "from paper_1903_05575_b200 import build; build.build(force=True)"; cp $SO /tmp/kc64.so
for v in r01 cur kc64 r01 cur; do
  cp /tmp/$v.so $SO
  python tools/f32_sizes.py | sed "s/^{/{\"v\": \"$v\", /" >> gpurun_out/r2j_sizes.jsonl 2>&1
  python bench.py --no-cpu --no-configs --no-sharded --no-e2e --no-parity --steps 5 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); v=d['variants']['c3_fp32']
print(json.dumps({'v': '$v', 'c3_fp32_tflops': v['value'], 'ms': v['ms_per_step'], 'clocks': v['clocks'], 'c3_f64': d['value']}))" >> gpurun_out/r2j_bench.jsonl
done
cp /tmp/cur.so $SO
