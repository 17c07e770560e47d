#!/bin/bash
# small kernels: split-K reduction buffers laid out [warp][component][lane] (conflict-free): parity + c1 A/B
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SO=paper_1903_05575_b200/libqgemm.so
cp _variants/small_new.so $SO
timeout 1200 python -m pytest tests -m gpu -q -x -k "small or tiny or c1 or ragged or exact_integer or randomized or graph or auto_policy" > gpurun_out/r2zi_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2zi_tests.log
for r in 1 2; do for v in small_old small_new; do
  cp _variants/$v.so $SO
  echo "== $v r$r" >> gpurun_out/r2zi_c1.txt
  timeout 300 python tools/c1_probe.py >> gpurun_out/r2zi_c1.txt 2>&1
done; done
cp _variants/small_new.so $SO
