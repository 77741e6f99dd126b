# Everything the round's evidence needs, in one GPU call:
#  - GPU test suite, smoke()
#  - bench lines: config 3 (default), reference arm, config 2 and config 4
#  - ncu launch list + one --set full capture of the config-3 fine sweep
#  - phase timing of the critical slice
TAG=${1:-r01}
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$TAG.txt 2>&1
python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
python bench.py --config 2 --steps 5 --warmup 3 > gpurun_out/bench_c2_$TAG.json 2> gpurun_out/bench_c2_$TAG.err
python bench.py --config 4 --steps 3 --warmup 3 > gpurun_out/bench_c4_$TAG.json 2> gpurun_out/bench_c4_$TAG.err
python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5_$TAG.json 2> gpurun_out/bench_c5_$TAG.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --dist --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_dist1_$TAG.json 2> gpurun_out/bench_dist1_$TAG.err
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-parareal"
$CMD > gpurun_out/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD > gpurun_out/ncu1_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_fine_sweep -c 1 -o gpurun_out/prof_$TAG $CMD > gpurun_out/ncu2_$TAG.log 2>&1
bash tools/phases.sh 3 > gpurun_out/phases_$TAG.txt 2>&1
python tools/slice_iters.py > gpurun_out/slices_$TAG.txt 2>&1
python tools/slice_finish.py > gpurun_out/finish_$TAG.txt 2>&1
echo done
