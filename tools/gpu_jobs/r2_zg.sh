#!/bin/bash
# host-streamed path: first chunk 64 k with a x4 ramp (QG_HOST_KC0_DIV 16, QG_HOST_RAMP 4) vs 256: parity + e2e A/B
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SO=paper_1903_05575_b200/libqgemm.so
cp _variants/host_new.so $SO
timeout 900 python -m pytest tests/test_gpu_host.py -m gpu -q -x > gpurun_out/r2zg_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2zg_tests.log
for r in 1 2 3; do for v in host_old host_new; do
  cp _variants/$v.so $SO
  timeout 600 python bench.py --no-cpu --no-configs --no-sharded --no-parity --steps 3 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']
print(json.dumps({'v': '$v', 'e2e_tflops': e['value'], 'e2e_ms': e['ms_per_step'], 'device_ms': d['ms_per_step']}))" >> gpurun_out/r2zg_e2e.jsonl
done; done
cp _variants/host_new.so $SO
