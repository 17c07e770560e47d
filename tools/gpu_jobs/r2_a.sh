#!/bin/bash
cd $GRAFT_REPO_ROOT
nproc > gpurun_out/r1_nproc.txt; free -g >> gpurun_out/r1_nproc.txt; nvidia-smi -L >> gpurun_out/r1_nproc.txt
timeout 2000 python -m pytest tests -m gpu -q -k "pack or qherk_lower or qherk_c4_full or c3_full or c5 or bench_contract or our_arm" > gpurun_out/r1_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r1_tests.log
timeout 600 python bench.py > gpurun_out/r1_bench.json 2> gpurun_out/r1_bench.err
echo "bench rc=$?" >> gpurun_out/r1_bench.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --debug-one-device --size 2048 --steps 2 --warmup 1 --no-e2e > gpurun_out/r1_dbg2.json 2> gpurun_out/r1_dbg2.err
echo "dbg rc=$?" >> gpurun_out/r1_dbg2.err
