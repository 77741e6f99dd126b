# config-4/5 sweep time and PCG iterations for each tools/variants/<name>.so in $1
LIB=paper_2510_11023_b200/libparafrac_b200.so
cp $LIB /tmp/lib_keep.so
for n in ${1//,/ }; do
  cp tools/variants/$n.so $LIB
  for c in 4 5; do
    echo "$n c$c $(python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-parareal 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["ms_per_step"],1), round(d["roofline"]["pcg_iterations_per_solve"],3))')"
  done
done
cp /tmp/lib_keep.so $LIB
