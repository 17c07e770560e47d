#!/bin/bash
# FP32 running-sum slots under a persisting-L2 access-policy window (QG_TC2_L2_PERSIST=1, opt-in):
# parity subset with it on, interleaved A/B timing, DRAM bytes per launch
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
QG_TC2_L2_PERSIST=1 timeout 1200 python -m pytest tests -m gpu -q -x -k "f32 or fp32 or precision or c3_full" > gpurun_out/r2zt_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2zt_tests.log
for r in 1 2 3; do for v in 0 1; do
  echo "== persist$v r$r" >> gpurun_out/r2zt_ab.txt
  QG_TC2_L2_PERSIST=$v timeout 300 python tools/f32_c3_time.py >> gpurun_out/r2zt_ab.txt 2>&1
done; done
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active"
for v in 0 1; do
  QG_TC2_L2_PERSIST=$v timeout 600 ncu --metrics $M --clock-control none -k regex:qgemm_tc32_2cta -c 1 --csv --log-file gpurun_out/r2zt_persist$v.csv python tools/prof_step.py --precision f32 > gpurun_out/r2zt_persist$v.log 2>&1
done
# FP64 headline unaffected by the carve-out? (same process: FP32 call first, then c3 FP64)
QG_TC2_L2_PERSIST=1 timeout 300 python tools/ab_quick.py --reps 2 > gpurun_out/r2zt_f64_after.txt 2>&1
