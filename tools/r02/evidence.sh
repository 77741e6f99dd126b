#!/bin/bash
# round-2 evidence run: bench lines (configs 3 default, 2, 4, 5 at P=512), reference arm,
# launch list + ncu of the main config-3 sweep launch
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-r02e}
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench_c3.json 2> gpurun_out/${TAG}_bench_c3.err
timeout 600 python bench.py --config 2 --steps 20 --warmup 5 > gpurun_out/${TAG}_bench_c2.json 2> gpurun_out/${TAG}_bench_c2.err
timeout 900 python bench.py --config 4 --steps 5 --warmup 3 > gpurun_out/${TAG}_bench_c4.json 2> gpurun_out/${TAG}_bench_c4.err
timeout 1500 python bench.py --config 5 --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_c5.json 2> gpurun_out/${TAG}_bench_c5.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err
CMD="python bench.py --steps 2 --warmup 3 --no-parareal --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size --clock-control none -c 30 --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fine_sweep -s 1 -c 1 -o gpurun_out/${TAG}_prof_main $CMD > gpurun_out/${TAG}_ncu2.log 2>&1
echo done
