LIB=paper_2510_11023_b200/libparafrac_b200.so
cp $LIB /tmp/keep.so
for v in tloc cur tloc cur; do cp tools/variants/$v.so $LIB; echo "== $v"; python bench.py --config 5 --steps 1 --warmup 1 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d["ms_per_step"], d["parareal"])'; done
cp /tmp/keep.so $LIB
