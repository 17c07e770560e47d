#!/bin/bash
# DRAM bytes / L2 hit rate / tensor pipe of the FP32 pair kernel at c3 with and without QG_TC2_SLOT_KEEP
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SO=paper_1903_05575_b200/libqgemm.so
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active"
for v in keep0 keep1; do
  cp _variants/$v.so $SO
  timeout 600 ncu --metrics $M --clock-control none -k regex:qgemm_tc32_2cta -c 1 --csv --log-file gpurun_out/r2zs_$v.csv python tools/prof_step.py --precision f32 > gpurun_out/r2zs_$v.log 2>&1
done
cp _variants/keep1.so $SO
