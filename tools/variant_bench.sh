# time bench.py (extra args $2..) for each tools/variants/<name>.so listed in $1 (comma-separated)
LIB=paper_2510_11023_b200/libparafrac_b200.so
cp $LIB /tmp/lib_keep.so
V=$1; shift
for n in ${V//,/ }; do
  cp tools/variants/$n.so $LIB
  echo "$n: $(python bench.py --no-cpu-baseline $* 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],3), "ms", (d.get("parareal") or {}).get("time_to_tol_s"))')"
done
cp /tmp/lib_keep.so $LIB
