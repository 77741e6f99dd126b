# --set full capture of the config-4 column kernel (PCG variant) + rows kernels
CMD="python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline --no-parareal"
$CMD > gpurun_out/plain_cols.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k2_ -s 400 -c 7 -o gpurun_out/prof_cols_$1 $CMD > gpurun_out/ncu_cols.log 2>&1
echo rc=$?
