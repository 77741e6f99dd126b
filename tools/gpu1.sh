set -x
python bench.py > gpurun_out/bench_r01.txt 2> gpurun_out/bench_r01.err
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-parareal"
$CMD > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu1.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_fine_sweep -c 1 -o gpurun_out/prof_fine $CMD > gpurun_out/ncu2.log 2>&1
echo done
