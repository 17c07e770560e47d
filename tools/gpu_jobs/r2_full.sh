#!/bin/bash
# full GPU suite (timed) + smoke
cd $GRAFT_REPO_ROOT
start=$(date +%s)
timeout 3000 python -m pytest tests -m gpu -q > gpurun_out/r2full_tests.log 2>&1
echo "rc=$? seconds=$(( $(date +%s) - start ))" >> gpurun_out/r2full_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2full_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2full_smoke.log
