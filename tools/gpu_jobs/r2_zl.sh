#!/bin/bash
# final evidence with the TMA-reduction ring epilogue (beta == 1) and the beta == 0 ring: full -m gpu suite, bench line, smoke,
# launch list of the bench command, c4 qgemm / QHERK metrics, full ncu of the c3 DMMA kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
start=$(date +%s)
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/r2zl_tests.log 2>&1
echo "rc=$? seconds=$(( $(date +%s) - start ))" >> gpurun_out/r2zl_tests.log
timeout 900 python bench.py > gpurun_out/r2zl_bench.json 2> gpurun_out/r2zl_bench.err; echo "bench rc=$?" >> gpurun_out/r2zl_bench.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2zl_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2zl_smoke.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2zl_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-configs --no-sharded > gpurun_out/r2zl_ncu_launch.log 2>&1
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__ops_path_tensor_src_fp64.sum"
timeout 600 ncu --metrics $M --clock-control none -k regex:qgemm_dmma -c 1 --csv python tools/prof_c4.py > gpurun_out/r2zl_c4_qgemm.csv 2>&1
timeout 600 ncu --metrics $M --clock-control none -k regex:qgemm_dmma -c 1 --csv python tools/prof_c4.py --herk > gpurun_out/r2zl_c4_qherk.csv 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:qgemm_dmma -c 1 -o gpurun_out/r2zl_c3 -f \
  python tools/prof_step.py > gpurun_out/r2zl_ncu_c3.log 2>&1
python tools/ncu_summary.py gpurun_out/r2zl_c3.ncu-rep > gpurun_out/r2zl_c3_summary.txt 2>&1
