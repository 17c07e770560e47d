#!/bin/bash
# tiny kernel: 8 vs 4 warps per CTA (c1 probe, PDL default), parity subset; FP32 accuracy vs K
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -m gpu -q -x -k "tiny or small" > gpurun_out/r2d_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2d_tests.log
python tools/c1_probe.py > gpurun_out/r2d_c1_w8.jsonl 2>&1
QG_SMALL_PDL=0 python tools/c1_probe.py > gpurun_out/r2d_c1_w8_pdl0.jsonl 2>&1
QG_SMALL_PDL=0 timeout 300 ncu --set full --import-source on --cache-control none --clock-control none \
  -k regex:qgemm_tiny --launch-skip 20 --launch-count 1 -o gpurun_out/r2d_c1_w8 -f python tools/c1_probe.py --ncu 40 \
  > gpurun_out/r2d_ncu.log 2>&1
python tools/f32_accuracy.py > gpurun_out/r2d_f32acc.jsonl 2>&1
QG_NVCC_EXTRA="-DQG_TINY_WARPS=4" python -c "from paper_1903_05575_b200 import build; build.build(force=True)"
python tools/c1_probe.py > gpurun_out/r2d_c1_w4.jsonl 2>&1
