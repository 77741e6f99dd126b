"""profiles/dram_config<N>.json from an ncu launch list (dram bytes per kernel):
the DRAM traffic of one sweep step = the sum over the kernels of one step
(slice-0 head-start launch + k_bracket_all + the main k_fine_sweep launch in
1-D; every kernel of one sweep in 2-D), averaged over the complete steps.

    python tools/dram_json.py gpurun_out/launches.csv 3 [first_kernel_id] [kernels_per_step] > profiles/dram_config3.json
"""
import csv
import json
import sys
from collections import defaultdict

path, cfg = sys.argv[1], int(sys.argv[2])
first = int(sys.argv[3]) if len(sys.argv) > 3 else 1
per = int(sys.argv[4]) if len(sys.argv) > 4 else 3
rows = list(csv.reader(open(path)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[hi]
d, names = defaultdict(dict), {}
for r in rows[hi + 1:]:
    i = int(r[h.index("ID")])
    names[i] = r[h.index("Kernel Name")].split("(")[0]
    d[i][r[h.index("Metric Name")]] = float(r[h.index("Metric Value")].replace(",", ""))
ids = sorted(k for k in d if k >= first)
steps = [ids[j:j + per] for j in range(0, len(ids) - per + 1, per)]
tot = [sum(d[k]["dram__bytes_read.sum"] + d[k]["dram__bytes_write.sum"] for k in s) for s in steps]
dom = max(steps[0], key=lambda k: d[k]["gpu__time_duration.sum"] * d[k].get("launch__grid_size", 1))
out = {"config": cfg, "dram_bytes_per_step": sum(tot) / len(tot), "steps_averaged": len(tot),
       "dominant_kernel": names[dom], "dominant_grid": d[dom].get("launch__grid_size"),
       "dominant_dram_bytes": d[dom]["dram__bytes_read.sum"] + d[dom]["dram__bytes_write.sum"],
       "dominant_ns_cold": d[dom]["gpu__time_duration.sum"],
       "per_kernel_first_step": [{"kernel": names[k], "grid": d[k].get("launch__grid_size"),
                                  "ns": d[k]["gpu__time_duration.sum"],
                                  "dram_bytes": d[k]["dram__bytes_read.sum"] + d[k]["dram__bytes_write.sum"]}
                                 for k in steps[0]],
       "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
                 f"(--clock-control none, serialised, cold) over {len(tot)} steps of bench.py --config {cfg}; {path}"}
print(json.dumps(out, indent=1))
