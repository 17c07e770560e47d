#!/bin/bash
# final tree final tree of round 2 (with the opt-in FP32 L2 window launch path): full -m gpu suite, default bench line (FP32 roofline per step), smoke
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
start=$(date +%s)
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2zu_tests.log 2>&1
echo "rc=$? seconds=$(( $(date +%s) - start ))" >> gpurun_out/r2zu_tests.log
timeout 900 python bench.py > gpurun_out/r2zu_bench.json 2> gpurun_out/r2zu_bench.err; echo "bench rc=$?" >> gpurun_out/r2zu_bench.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2zu_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2zu_smoke.log
