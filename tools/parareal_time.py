import sys, time, numpy as np
sys.path.insert(0, "/root/repo")
import paper_2510_11023_b200 as pfb
from paper_2510_11023_b200 import _lib
for cfg in (3, 2):
    c = pfb.problems.CONFIGS[cfg]
    prob = pfb.config_problem(cfg); op = pfb.build_sine_operator(c["modes"]); g = pfb.TimeGrids(c["t_final"], c["nt"], c["m"])
    pfb.parareal_solve(prob, op, g, tol=c["tol"], k_max=c["nt"] + 1)
    for rep in range(2):
        t0 = time.perf_counter(); it, r = pfb.parareal_solve(prob, op, g, tol=c["tol"], k_max=c["nt"] + 1); t1 = time.perf_counter()
        print(f"cfg{cfg}: time-to-tol {t1-t0:.4f} s, {r.iterations} it, iteration_times {np.round(np.diff([0]+r.iteration_times), 4)}, stats {r.device_stats}")
