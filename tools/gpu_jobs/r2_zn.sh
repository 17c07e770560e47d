#!/bin/bash
# launch list of the bench command, the library's kernels only (r2_zl's unfiltered list
# ran out of its 400-launch budget on the device input generator's torch kernels)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'qgemm|tc2_|pack_kernel|pack_tc32' -c 400 --csv \
  --log-file gpurun_out/r2zn_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu > gpurun_out/r2zn_ncu_launch.log 2>&1
echo "rc=$?" >> gpurun_out/r2zn_ncu_launch.log
