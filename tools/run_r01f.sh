timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_r01f.txt 2>&1
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --dist --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_dist1.json 2> gpurun_out/bench_dist1.err
timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4_r01f.json 2> gpurun_out/bench_c4_r01f.err
timeout 900 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c5_r01f.json 2> gpurun_out/bench_c5_r01f.err
echo done
