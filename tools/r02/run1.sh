#!/bin/bash
# round-2 GPU call: tests, bench (config 3), launch list with DRAM bytes per kernel, full capture of the main sweep launch
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi -L > gpurun_out/smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
CMD="python bench.py --steps 2 --warmup 3 --no-parareal --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size --clock-control none -c 30 --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fine_sweep -s 1 -c 1 -o gpurun_out/prof_main $CMD > gpurun_out/ncu2.log 2>&1
echo done
