#!/bin/bash
# final tree: forced-remote-C epilogue parity (child process), N > 1 bench paths on one
# device (2 ranks), reference arm
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "remote_c_epilogue" > gpurun_out/r2zo_tests_remote.log 2>&1
echo "rc=$?" >> gpurun_out/r2zo_tests_remote.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 2 --debug-one-device --size 2048 --steps 2 --warmup 1 --no-e2e > gpurun_out/r2zo_bench_debug2.json 2> gpurun_out/r2zo_bench_debug2.err
echo "debug rc=$?" >> gpurun_out/r2zo_bench_debug2.err
timeout 600 python bench.py --impl reference > gpurun_out/r2zo_bench_ref.json 2> gpurun_out/r2zo_bench_ref.err
echo "ref rc=$?" >> gpurun_out/r2zo_bench_ref.err
