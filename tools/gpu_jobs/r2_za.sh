#!/bin/bash
# phase trace of the store-warp ring epilogue: c4 (K = 256), c3, c2
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SO=paper_1903_05575_b200/libqgemm.so
cp $SO /tmp/default.so
cp _variants/trace.so $SO
timeout 300 python tools/trace_phases.py --n 32768 --k 256 --ops NH --beta 1 > gpurun_out/r2za_trace.txt 2>&1
timeout 300 python tools/trace_phases.py --n 32768 --k 256 --ops NH --beta 0 >> gpurun_out/r2za_trace.txt 2>&1
timeout 300 python tools/trace_phases.py --n 8192 --k 8192 --ops NH --beta 1 >> gpurun_out/r2za_trace.txt 2>&1
timeout 300 python tools/trace_phases.py --n 1024 --ops NN --beta -0.5 >> gpurun_out/r2za_trace.txt 2>&1
cp /tmp/default.so $SO
