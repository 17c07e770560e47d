#!/bin/bash
# c1 latency probe (PDL off/on), ncu of the c1 kernel, FP32 c3 Freivalds test
cd $GRAFT_REPO_ROOT
QG_SMALL_PDL=0 python tools/c1_probe.py > gpurun_out/r2b_c1_pdl0.jsonl 2>&1
QG_SMALL_PDL=1 python tools/c1_probe.py > gpurun_out/r2b_c1_pdl1.jsonl 2>&1
QG_SMALL_PDL=0 timeout 300 ncu --set full --import-source on --cache-control none --clock-control none \
  -k regex:qgemm_small --launch-skip 20 --launch-count 1 -o gpurun_out/r2b_c1 -f python tools/c1_probe.py --ncu 40 \
  > gpurun_out/r2b_ncu.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -k "c3_full or quick_returns" > gpurun_out/r2b_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2b_tests.log
