#!/bin/bash
# FP32 running-sum slots kept in L2 (QG_TC2_SLOT_KEEP: evict_last policy on the slot's stores and
# reductions): FP32 parity tests with the new build, interleaved A/B timing, DRAM bytes per launch
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SO=paper_1903_05575_b200/libqgemm.so
cp _variants/keep1.so $SO
timeout 1200 python -m pytest tests -m gpu -q -x -k "f32 or fp32 or precision or c3_full" > gpurun_out/r2zr_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2zr_tests.log
for r in 1 2 3; do for v in keep0 keep1; do
  cp _variants/$v.so $SO
  echo "== $v r$r" >> gpurun_out/r2zr_ab.txt
  timeout 300 python tools/f32_c3_time.py >> gpurun_out/r2zr_ab.txt 2>&1
done; done
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active"
for v in keep0 keep1; do
  cp _variants/$v.so $SO
  echo "== $v" >> gpurun_out/r2zr_ncu.txt
  timeout 600 ncu --metrics $M --clock-control none -k regex:qgemm_tc32_2cta -c 1 --csv python tools/prof_step.py --precision f32 2>&1 | grep -v "^==" | cut -d, -f5,13,14,15 >> gpurun_out/r2zr_ncu.txt
done
cp _variants/keep1.so $SO
