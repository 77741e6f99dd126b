set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r01e.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_r01e.txt 2>&1
python bench.py > gpurun_out/bench_r01e.json 2> gpurun_out/bench_r01e.err
python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5_r01e.json 2> gpurun_out/bench_c5_r01e.err
echo done
