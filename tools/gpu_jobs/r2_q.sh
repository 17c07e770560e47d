#!/bin/bash
# round-2 evidence: full bench line, reference arm, 2-rank debug, launch list, full ncu of the top kernel
cd $GRAFT_REPO_ROOT
python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02_bench_ref.json 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 \
  bench.py --gpus 2 --debug-one-device --size 2048 --steps 2 --warmup 1 --no-e2e > gpurun_out/r02_bench_debug2.json 2> gpurun_out/r02_bench_debug2.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r02_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/r02_ncu_launch_run.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:qgemm_dmma --launch-skip 1 --launch-count 1 \
  -o gpurun_out/r02_c3_dmma -f python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e --no-f32 --no-configs --no-sharded --no-parity \
  > gpurun_out/r02_ncu_full.log 2>&1
