#!/bin/bash
# beta == 1 ring epilogue by TMA reductions (QG_C_REDUCE): new test first, full suite, then A/B
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SO=paper_1903_05575_b200/libqgemm.so
cp _variants/cr1.so $SO
timeout 600 python -m pytest tests -m gpu -q -x -k "beta_one_tma_reduction" > gpurun_out/r2zk_tests_new.log 2>&1
echo "rc=$?" >> gpurun_out/r2zk_tests_new.log
for r in 1 2; do for v in cr0 cr1; do
  cp _variants/$v.so $SO
  echo "== $v r$r" >> gpurun_out/r2zk_ab.txt
  timeout 300 python tools/ab_quick.py --reps 3 >> gpurun_out/r2zk_ab.txt 2>&1
  timeout 300 python tools/c4_time.py --tag $v >> gpurun_out/r2zk_ab.txt 2>&1
done; done
cp _variants/cr1.so $SO
start=$(date +%s)
timeout 2000 python -m pytest tests -m gpu -q -x > gpurun_out/r2zk_tests.log 2>&1
echo "rc=$? seconds=$(( $(date +%s) - start ))" >> gpurun_out/r2zk_tests.log
