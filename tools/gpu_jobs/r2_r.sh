#!/bin/bash
# launch list of the library's kernels in the default bench command
cd $GRAFT_REPO_ROOT
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"qgemm|tc2_|pack_kernel|pack_tc32" -c 400 --csv \
  --log-file gpurun_out/r02_launches_lib.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/r02_ncu_launch_lib.log 2>&1
