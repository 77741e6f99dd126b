python tools/coarse2d_time.py 128
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2d.csv python tools/coarse2d_time.py 8 > /dev/null 2>&1
python - << 'PY'
import csv, collections
lines = open('gpurun_out/launches_c2d.csv').read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.reader(lines[start:]))
h = rows[0]; ki = h.index('Kernel Name'); vi = h.index('Metric Value')
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    k = r[ki].split('(')[0]; agg[k][0] += 1; agg[k][1] += float(r[vi].replace(',', ''))
tot = sum(v[1] for v in agg.values())
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{t/1e6:9.2f} ms {100*t/tot:5.1f}%  n={n:6d}  avg {t/n/1e3:8.1f} us  {k[:70]}")
print("total kernel ms", tot/1e6)
PY
