"""2-D parareal time-to-tol with the per-iteration split (fine sweep vs coarse correction).

    python tools/parareal_time2d.py 4 [k_max]
"""
import sys, time, numpy as np
sys.path.insert(0, "/root/repo")
import paper_2510_11023_b200 as pfb
from paper_2510_11023_b200 import _lib
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
kmax = int(sys.argv[2]) if len(sys.argv) > 2 else None
c = pfb.problems.CONFIGS[cfg]
prob = pfb.config_problem(cfg)
op = pfb.build_sine_operator(c["modes"], dims=2)
g = pfb.TimeGrids(c["t_final"], c["nt"], c["m"])
t0 = time.perf_counter(); tr = pfb.run_coarse(prob, op, g); t1 = time.perf_counter()
print(f"cfg{cfg}: run_coarse {t1 - t0:.3f} s")
t0 = time.perf_counter()
it, r = pfb.parareal_solve(prob, op, g, tol=c["tol"], k_max=kmax or c["nt"] + 1)
t1 = time.perf_counter()
print(f"cfg{cfg}: time-to-tol {t1 - t0:.3f} s, {r.iterations} it ({r.stop_reason}), diffs {np.array(r.diffs)}")
print("iteration times", np.round(np.diff([0] + list(r.iteration_times)), 4))
print("stats", r.device_stats)
