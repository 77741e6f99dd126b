# bench + slice finish spread for each tools/variants/<name>.so in $1
LIB=paper_2510_11023_b200/libparafrac_b200.so
cp $LIB /tmp/lib_keep.so
for n in ${1//,/ }; do
  cp tools/variants/$n.so $LIB
  echo "== $n: $(python bench.py --no-cpu-baseline --steps 10 --warmup 3 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],3), "ms", (d.get("parareal") or {}).get("time_to_tol_s"))')"
  python tools/slice_finish.py 2>&1 | head -3
done
cp /tmp/lib_keep.so $LIB
