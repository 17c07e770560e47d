#!/bin/bash
# FP32 A/B on one box: direct feed (auto) vs packed (policy 1), twice
cd $GRAFT_REPO_ROOT
for pol in 0 1 0 1; do
  python bench.py --no-cpu --no-configs --no-sharded --no-e2e --no-parity --steps 5 --policy $pol 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); v=d['variants']['c3_fp32']
print(json.dumps({'policy': $pol, 'c3_fp32_tflops': v['value'], 'ms': v['ms_per_step'], 'clocks': v['clocks'], 'launches': v['launches_per_step'], 'f64': d['value']}))" >> gpurun_out/r2p_bench.jsonl
done
ncu --metrics gpu__time_duration.sum,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio --clock-control none -k regex:tc32_2cta -c 2 --csv python bench.py --no-cpu --no-configs --no-sharded --no-e2e --no-parity --steps 1 --warmup 0 > gpurun_out/r2p_ncu_direct.csv 2>&1
ncu --metrics gpu__time_duration.sum,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum --clock-control none -k regex:tc32_2cta -c 2 --csv python bench.py --no-cpu --no-configs --no-sharded --no-e2e --no-parity --steps 1 --warmup 0 --policy 1 > gpurun_out/r2p_ncu_packed.csv 2>&1
