# 2-D PCG batch size sweep (PF_CHUNK2D) for configs 4 and 5
for cfg in 4 5; do
  for ch in 0 64 32 16 8; do
    echo "config $cfg chunk $ch: $(PF_CHUNK2D=$ch python bench.py --config $cfg --steps 2 --warmup 1 --no-cpu-baseline --no-parareal 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],1), "ms", d["roofline"]["pcg_iterations_per_solve"])')"
  done
done
