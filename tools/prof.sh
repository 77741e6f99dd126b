# usage: bash tools/prof.sh TAG  -> gpu_check, bench line, ncu full capture of the fine sweep
TAG=${1:-x}
python tools/gpu_check.py > gpurun_out/gpu_check_$TAG.txt 2>&1
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-parareal"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_fine_sweep -c 1 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu_$TAG.log 2>&1
echo done
