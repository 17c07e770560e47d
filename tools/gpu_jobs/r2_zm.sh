#!/bin/bash
# beta == 0 tiles through the ring epilogue (QG_RING_BETA0): new test, ring tests, then A/B
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SO=paper_1903_05575_b200/libqgemm.so
cp _variants/rb1.so $SO
timeout 900 python -m pytest tests -m gpu -q -x -k "ring or beta or c1_full or c5 or nan" > gpurun_out/r2zm_tests_new.log 2>&1
echo "rc=$?" >> gpurun_out/r2zm_tests_new.log
for r in 1 2; do for v in rb0 rb1; do
  cp _variants/$v.so $SO
  echo "== $v r$r" >> gpurun_out/r2zm_ab.txt
  timeout 300 python tools/ab_quick.py --reps 3 >> gpurun_out/r2zm_ab.txt 2>&1
done; done
cp _variants/rb1.so $SO
