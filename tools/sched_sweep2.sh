for s in "5,16,7,64,6,128,5,256,4" "5,16,7,48,6,128,5,256,4" "5,16,7,64,6,128,5,192,4" "5,16,7,64,5,256,4" "5,12,7,64,6,128,5,256,4" "6,16,7,64,6,128,5,256,4"; do
  echo "$s: $(PF_EXT_SCHED=$s python bench.py --no-cpu-baseline --no-parareal --steps 10 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],3), "ms", round(d["roofline"]["pcg_iterations_per_solve"],4))')"
done
