CMD="python bench.py --config 4 --steps 1 --warmup 1 --no-cpu-baseline --no-parareal"
$CMD > gpurun_out/plain2d.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches2d.csv $CMD > gpurun_out/ncu2d.log 2>&1
python - << 'PY'
import csv, collections
lines = open('gpurun_out/launches2d.csv').read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.reader(lines[start:]))
h = rows[0]; ki = h.index('Kernel Name'); vi = h.index('Metric Value')
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    k = r[ki].split('(')[0]
    agg[k][0] += 1; agg[k][1] += float(r[vi].replace(',', ''))
tot = sum(v[1] for v in agg.values())
with open('gpurun_out/prof2d_summary.txt', 'w') as f:
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        line = f"{t/1e6:9.1f} ms {100*t/tot:5.1f}%  n={n:6d}  avg {t/n/1e3:8.1f} us  {k[:90]}"
        print(line); f.write(line + "\n")
PY
