#!/bin/bash
# epilogue skew sweep: c4 qgemm / qherk, c3 unaffected
cd $GRAFT_REPO_ROOT
for ns in 0 2000 4000 6000 10000; do
  QG_NVCC_EXTRA="-DQG_EPI_SKEW_NS=$ns" python -c "from paper_1903_05575_b200 import build; build.build(force=True)"
  python tools/c4_time.py --tag skew$ns >> gpurun_out/r2s_c4.jsonl 2>&1
done
