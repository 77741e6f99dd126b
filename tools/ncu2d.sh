# one --set full capture of a run of consecutive 2-D kernels (a full PCG iteration) at config ${1:-4}
CFG=${1:-4}
CMD="python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline --no-parareal"
$CMD > gpurun_out/plain2d_full.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k2_ -s 400 -c 14 -o gpurun_out/prof2d_c$CFG $CMD > gpurun_out/ncu2d_full.log 2>&1
echo rc=$?
