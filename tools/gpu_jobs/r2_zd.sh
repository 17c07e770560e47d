#!/bin/bash
# half-k-tile ring (6 stages of 8 k): full suite, then A/B against the 3-stage build
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SO=paper_1903_05575_b200/libqgemm.so
cp _variants/half_stage.so $SO
start=$(date +%s)
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/r2zd_tests.log 2>&1
echo "rc=$? seconds=$(( $(date +%s) - start ))" >> gpurun_out/r2zd_tests.log
for r in 1 2; do
for v in full_stage half_stage; do
  cp _variants/$v.so $SO
  echo "== $v r$r" >> gpurun_out/r2zd_ab.txt
  timeout 300 python tools/ab_quick.py --reps 3 >> gpurun_out/r2zd_ab.txt 2>&1
  timeout 300 python tools/c4_time.py --tag $v >> gpurun_out/r2zd_ab.txt 2>&1
done
done
cp _variants/half_stage.so $SO
cp _variants/trace_half.so $SO
timeout 300 python tools/trace_phases.py --n 32768 --k 256 --ops NH --beta 1 > gpurun_out/r2zd_trace.txt 2>&1
cp _variants/half_stage.so $SO
