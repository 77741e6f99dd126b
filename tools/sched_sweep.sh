# 1-D config-3 sweep / time-to-tol for guess-order schedules of the first slice (PF_EXT_SCHED)
for s in "5,16,7,64,6,128,5,256,4" "5,16,7,32,6,64,5,128,4" "5,16,7,128,6,256,5,512,4" "5,16,7,64,6,256,5" "5,8,7,64,6,128,5,256,4" "4,16,7,64,6,128,5,256,4"; do
  echo "$s: $(PF_EXT_SCHED=$s python bench.py --no-cpu-baseline --steps 10 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],3), "ms", round(d["roofline"]["pcg_iterations_per_solve"],4), (d.get("parareal") or {}).get("time_to_tol_s"))')"
done
