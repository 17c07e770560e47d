#!/bin/bash
# FP32: per-component chunk commits (drain overlaps the tail MMAs): speed kc 32 vs off, FP32 tests
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x -k "f32 or tc32 or split" > gpurun_out/r2i_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2i_tests.log
python tools/f32_sizes.py | sed 's/^{/{"kc": 32, /' > gpurun_out/r2i_sizes.jsonl 2>&1
python bench.py --no-cpu --no-configs --no-sharded --no-e2e --no-parity --steps 5 > gpurun_out/r2i_bench_kc32.json 2>/dev/null
QG_NVCC_EXTRA="-DQG_TC2_CHUNK_KT=100000" python -c "from paper_1903_05575_b200 import build; build.build(force=True)"
python tools/f32_sizes.py | sed 's/^{/{"kc": 100000, /' >> gpurun_out/r2i_sizes.jsonl 2>&1
python bench.py --no-cpu --no-configs --no-sharded --no-e2e --no-parity --steps 5 > gpurun_out/r2i_bench_kcoff.json 2>/dev/null
