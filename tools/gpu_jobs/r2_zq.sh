#!/bin/bash
# final tree: full ncu of the FP32 pair kernel at c3 (chunked accumulation + L2 reductions; the
# committed FP32 capture is round 1's), of c2 (1024^3 N/N) and of the pack kernels
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/prof_step.py --precision f32 > gpurun_out/r2zq_f32_plain.log 2>&1; echo "rc=$?" >> gpurun_out/r2zq_f32_plain.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:qgemm_tc32_2cta -c 1 -o gpurun_out/r2zq_f32 -f \
  python tools/prof_step.py --precision f32 > gpurun_out/r2zq_ncu_f32.log 2>&1
python tools/ncu_summary.py gpurun_out/r2zq_f32.ncu-rep > gpurun_out/r2zq_f32_summary.txt 2>&1
ncu -i gpurun_out/r2zq_f32.ncu-rep --page raw --csv > gpurun_out/r2zq_f32_raw.csv 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 20 --csv \
  --log-file gpurun_out/r2zq_f32_launches.csv python tools/prof_step.py --precision f32 > gpurun_out/r2zq_f32_launches.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:qgemm_dmma -c 1 -o gpurun_out/r2zq_c2 -f \
  python tools/prof_step.py --n 1024 --ops NN > gpurun_out/r2zq_ncu_c2.log 2>&1
python tools/ncu_summary.py gpurun_out/r2zq_c2.ncu-rep > gpurun_out/r2zq_c2_summary.txt 2>&1
rm -f gpurun_out/r2zq_c2.ncu-rep
