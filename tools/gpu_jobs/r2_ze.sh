#!/bin/bash
# L2 prefetch of ring-epilogue C tiles (QG_RING_C_PREFETCH_KT) and of the next unit's first k-tile (QG_NEXT_PREFETCH_KT)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SO=paper_1903_05575_b200/libqgemm.so
cp _variants/pf_both.so $SO
timeout 1500 python -m pytest tests -m gpu -q -x -k "ring or qherk or group4 or c2_all or c4_full or concurrent or graph or randomized or short_k" > gpurun_out/r2ze_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2ze_tests.log
for r in 1 2; do
for v in pf_off pf_c pf_n pf_both; do
  cp _variants/$v.so $SO
  echo "== $v r$r" >> gpurun_out/r2ze_ab.txt
  timeout 300 python tools/ab_quick.py --reps 3 >> gpurun_out/r2ze_ab.txt 2>&1
  timeout 300 python tools/c4_time.py --tag $v >> gpurun_out/r2ze_ab.txt 2>&1
done
done
cp _variants/pf_both.so $SO
