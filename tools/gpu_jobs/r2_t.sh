#!/bin/bash
# c4 per-lane epilogue: 256-bit C stores / loads (A/B builds)
cd $GRAFT_REPO_ROOT
for f in "" "-DQG_C_ST256=1" "-DQG_C_ST256=1 -DQG_C_LD256=1" "-DQG_C_LD256=1"; do
  QG_NVCC_EXTRA="$f" python -c "from paper_1903_05575_b200 import build; build.build(force=True)"
  python tools/c4_time.py --tag "$f" >> gpurun_out/r2t_c4.jsonl 2>&1
done
QG_NVCC_EXTRA="-DQG_C_ST256=1" python -c "from paper_1903_05575_b200 import build; build.build(force=True)"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active --clock-control none -k regex:qgemm_dmma -c 2 --csv python tools/c4_time.py --tag ncu > gpurun_out/r2t_ncu_st256.csv 2>&1
QG_NVCC_EXTRA="" python -c "from paper_1903_05575_b200 import build; build.build(force=True)"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active --clock-control none -k regex:qgemm_dmma -c 2 --csv python tools/c4_time.py --tag ncu > gpurun_out/r2t_ncu_base.csv 2>&1
