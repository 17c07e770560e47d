#!/bin/bash
# store-warp ring epilogue (QG_C_STORE_WARP) + FP32 remainder split: parity, then A/B
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SO=paper_1903_05575_b200/libqgemm.so
cp $SO /tmp/default.so
timeout 1500 python -m pytest tests -m gpu -q -x -k "ring or qherk or remainder or f32_split or group4 or c2_all or concurrent or graph or randomized" > gpurun_out/r2w_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2w_tests.log
for r in 1 2; do
for v in sw0 sw1 sw1_kt1 sw0_kt1; do
  cp _variants/$v.so $SO
  echo "== $v r$r" >> gpurun_out/r2w_ab.txt
  timeout 300 python tools/ab_quick.py --reps 3 >> gpurun_out/r2w_ab.txt 2>&1
  timeout 300 python tools/c4_time.py --tag $v >> gpurun_out/r2w_ab.txt 2>&1
done
done
cp /tmp/default.so $SO
timeout 300 python tools/f32_sizes.py > gpurun_out/r2w_f32_sizes.jsonl 2>&1
QG_TC2_S=1 timeout 300 python tools/f32_sizes.py > gpurun_out/r2w_f32_sizes_s1.jsonl 2>&1
