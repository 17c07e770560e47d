#!/bin/bash
# tile-exact small kernel with 8 warps per CTA (QG_TINY_WARPS=8) now that the reduction is conflict-free
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SO=paper_1903_05575_b200/libqgemm.so
cp _variants/tiny8.so $SO
timeout 900 python -m pytest tests -m gpu -q -x -k "tiny or c1" > gpurun_out/r2zj_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2zj_tests.log
for r in 1 2; do for v in small_new tiny8; do
  cp _variants/$v.so $SO
  echo "== $v r$r" >> gpurun_out/r2zj_c1.txt
  timeout 300 python tools/c1_probe.py >> gpurun_out/r2zj_c1.txt 2>&1
done; done
cp _variants/small_new.so $SO
