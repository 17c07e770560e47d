#!/bin/bash
# tiny (tile-exact) small kernel: parity, c1 latency with PDL 0/1/2, ncu of the c1 kernel
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x -k "tiny or small or c1 or auto_policy or graph or concurrent" > gpurun_out/r2c_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2c_tests.log
for m in 0 1 2; do QG_SMALL_PDL=$m python tools/c1_probe.py > gpurun_out/r2c_c1_pdl$m.jsonl 2>&1; done
QG_SMALL_PDL=0 timeout 300 ncu --set full --import-source on --cache-control none --clock-control none \
  -k regex:qgemm_tiny --launch-skip 20 --launch-count 1 -o gpurun_out/r2c_c1 -f python tools/c1_probe.py --ncu 40 \
  > gpurun_out/r2c_ncu.log 2>&1
