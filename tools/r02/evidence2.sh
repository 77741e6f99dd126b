#!/bin/bash
# round-2 final evidence (one GPU call): smoke, GPU tests, bench lines (configs 3, 2, 4, 5 at P = 512),
# the reference arm, ncu launch list + full capture of the main sweep launch, per-warp timeline and
# whole-sweep substep durations (default engine and the DFMA helper), microbenchmarks.
#   here first:  tools/r02/evidence2.sh build     (trace variants + microbenchmarks, cross-compiled)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
if [ "$1" = "build" ]; then
  (TRACE_SO=trace_s1 bash tools/r02/trace.sh build) & (TRACE_SO=trace_s0 bash tools/r02/trace.sh build -DPF_TRACE_SLICE=0) &
  (TRACE_SO=trace_noside bash tools/r02/trace.sh build -DPF_NO_SIDE) &
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/fft10_bench.bin tools/fft10_bench.cu &
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/tanh_bench.bin tools/tanh_bench.cu &
  wait; exit 0
fi
mkdir -p gpurun_out
TAG=${1:-r02c}
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest_gpu.txt 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench_c3.json 2> gpurun_out/${TAG}_bench_c3.err
timeout 600 python bench.py --config 2 --steps 20 --warmup 5 > gpurun_out/${TAG}_bench_c2.json 2> gpurun_out/${TAG}_bench_c2.err
timeout 900 python bench.py --config 4 --steps 5 --warmup 3 > gpurun_out/${TAG}_bench_c4.json 2> gpurun_out/${TAG}_bench_c4.err
timeout 1500 python bench.py --config 5 --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_c5.json 2> gpurun_out/${TAG}_bench_c5.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/${TAG}_bench_ref.json 2> gpurun_out/${TAG}_bench_ref.err
CMD="python bench.py --steps 2 --warmup 3 --no-parareal --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size --clock-control none -c 30 --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fine_sweep -s 1 -c 1 -o gpurun_out/${TAG}_prof_main $CMD > gpurun_out/${TAG}_ncu2.log 2>&1
for v in trace_s1 trace_s0 trace_noside; do
  echo "=== $v (default far-history engine)"; TRACE_SO=$v timeout 120 bash tools/r02/trace.sh 3 2>&1
done > gpurun_out/${TAG}_trace.txt
for v in trace_s1; do
  echo "=== $v PF_FAR_TC=0 (DFMA helper, one pass per tile)"; PF_FAR_TC=0 TRACE_SO=$v timeout 120 bash tools/r02/trace.sh 3 2>&1 | tail -n 32
done > gpurun_out/${TAG}_trace_dfma_helper.txt
for tc in 0 1 2; do echo "PF_FAR_TC=$tc: $(PF_FAR_TC=$tc python bench.py --no-cpu-baseline --no-parareal 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],3), "ms per sweep")')"; done > gpurun_out/${TAG}_far_history_engines.txt 2>&1
bash tools/r02/early_phase.sh trace_s0 > gpurun_out/${TAG}_early_phase_slice0.txt 2>&1
python tools/slice_finish.py > gpurun_out/${TAG}_slice_finish.txt 2>&1
(./tools/fft10_bench.bin; ./tools/tanh_bench.bin) > gpurun_out/${TAG}_microbench.txt 2>&1
echo done
