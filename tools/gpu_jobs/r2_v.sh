#!/bin/bash
# round-2 re-entry check: full GPU suite, smoke, default bench line
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
start=$(date +%s)
timeout 3000 python -m pytest tests -m gpu -q -x > gpurun_out/r2v_tests.log 2>&1
echo "rc=$? seconds=$(( $(date +%s) - start ))" >> gpurun_out/r2v_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2v_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2v_smoke.log
timeout 900 python bench.py > gpurun_out/r2v_bench.json 2> gpurun_out/r2v_bench.err; echo "bench rc=$?" >> gpurun_out/r2v_bench.err
