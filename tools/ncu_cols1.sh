# --set full capture of the config-4 column setup kernel (k2_cols16<true>)
CMD="python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline --no-parareal"
$CMD > gpurun_out/plain_cols1.log 2>&1 && \
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:k2_cols16<.bool.1, .int.16" -s 20 -c 1 -o gpurun_out/prof_cols1 $CMD > gpurun_out/ncu_cols1.log 2>&1
echo rc=$?
