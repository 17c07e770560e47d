#!/bin/bash
# ring epilogue at every K + early slot release (QG_EARLY_RELEASE): full suite, then A/B
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SO=paper_1903_05575_b200/libqgemm.so
cp _variants/er1.so $SO
start=$(date +%s)
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2y_tests.log 2>&1
echo "rc=$? seconds=$(( $(date +%s) - start ))" >> gpurun_out/r2y_tests.log
for r in 1 2; do
for v in er0 er1; do
  cp _variants/$v.so $SO
  echo "== $v r$r" >> gpurun_out/r2y_ab.txt
  timeout 300 python tools/ab_quick.py --reps 3 >> gpurun_out/r2y_ab.txt 2>&1
  timeout 300 python tools/c4_time.py --tag $v >> gpurun_out/r2y_ab.txt 2>&1
done
done
cp _variants/er1.so $SO
