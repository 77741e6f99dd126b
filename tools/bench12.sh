for c in 1 2; do python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null > gpurun_out/b$c.json; python -c "import json; d=json.load(open('gpurun_out/b$c.json')); print($c, d['ms_per_step'], d['value'], d['parareal']['time_to_tol_s'])"; done
timeout 600 python -m pytest tests -m gpu -q 2>&1 | tail -2
