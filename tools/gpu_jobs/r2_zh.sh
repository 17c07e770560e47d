#!/bin/bash
# final tree: full -m gpu suite, smoke, bench line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
start=$(date +%s)
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2zh_tests.log 2>&1
echo "rc=$? seconds=$(( $(date +%s) - start ))" >> gpurun_out/r2zh_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2zh_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2zh_smoke.log
timeout 900 python bench.py > gpurun_out/r2zh_bench.json 2> gpurun_out/r2zh_bench.err; echo "bench rc=$?" >> gpurun_out/r2zh_bench.err
