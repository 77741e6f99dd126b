"""Sweep time and PCG iterations of the config-3 sweep under guess-order schedules (PF_EXT_SCHED:
order,until,order,until,...,order for the tau-extrapolation table; one process per schedule)."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
CODE = """
import sys, numpy as np
sys.path.insert(0, {root!r})
import paper_2510_11023_b200 as p
from paper_2510_11023_b200 import _lib
pr = p.config_problem(3); op = p.build_sine_operator(512); g = p.TimeGrids(2.0, 64, 1024)
t = p.run_coarse(pr, op, g)
ctx = _lib.context_for(pr, op, g)
best = 1e9
for i in range(4):
    ctx.reset_stats() if hasattr(ctx, "reset_stats") else None
    out = p.fine_sweep_intervals(t, 0, 64, op, g, pr)
    s = ctx.stats()
    best = min(best, s["last_fine_ms"])
print(round(best, 3), "ms", s)
"""
scheds = sys.argv[1:] or ["5,16,7,64,6,128,5,256,4"]
for sc in scheds:
    r = subprocess.run([sys.executable, "-c", CODE.format(root=ROOT)], capture_output=True, text=True,
                       env=dict(os.environ, PF_EXT_SCHED=sc))
    print(f"{sc:36s} {r.stdout.strip()[:120]} {r.stderr.strip()[-200:]}")
