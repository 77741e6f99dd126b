"""PCG iterations and device time per slice of the config-3 sweep (load balance diagnostic)."""
import sys, numpy as np
sys.path.insert(0, "/root/repo")
import paper_2510_11023_b200 as pfb
from paper_2510_11023_b200 import _lib
c = pfb.problems.CONFIGS[3]
prob = pfb.config_problem(3); op = pfb.build_sine_operator(512); g = pfb.TimeGrids(2.0, 64, 1024)
tr = pfb.run_coarse(prob, op, g)
ctx = _lib.context_for(prob, op, g)
pfb.fine_sweep_intervals(tr, 0, 64, op, g, prob)
rows = []
for n in range(64):
    s0 = ctx.stats()
    pfb.fine_sweep_intervals(tr, n, n + 1, op, g, prob)
    s1 = ctx.stats()
    rows.append((n, (s1["pcg_iterations"] - s0["pcg_iterations"]) / 1024, s1["last_fine_ms"]))
for n, it, ms in rows[:6] + rows[-3:]:
    print(f"slice {n:2d}: {it:.3f} CG it/solve, {ms:.2f} ms alone")
its = np.array([r[1] for r in rows]); ms = np.array([r[2] for r in rows])
print("mean it", its.mean(), "max it", its.max(), "mean ms", ms.mean(), "max ms", ms.max())
