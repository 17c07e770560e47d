#!/bin/bash
# FP32 direct feed (no pack): parity of every FP32 path, speed vs packed (A/B)
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -q -x -k "f32 or tc32 or split or host or randomized or graph" > gpurun_out/r2o_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2o_tests.log
python bench.py --no-cpu --no-configs --no-sharded --no-e2e --no-parity --steps 5 2>/dev/null > gpurun_out/r2o_bench_direct.json
QG_POLICY=1 python - > gpurun_out/r2o_bench_packed.json 2>&1 <<'PY'
import json, subprocess, sys
PY
python tools/f32_sizes.py > gpurun_out/r2o_sizes_direct.jsonl 2>&1
