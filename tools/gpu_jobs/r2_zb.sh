#!/bin/bash
# new short-K ring test; launch list of the bench command (library kernels only)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "short_k_stream_k or ring_epilogue_edges" > gpurun_out/r2zb_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2zb_tests.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'qgemm|tc2_|pack_kernel|pack_tc32' -c 400 --csv \
  --log-file gpurun_out/r2zb_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/r2zb_ncu_launch.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r2zb_ncu_launch.log
