"""Time-to-tol of parareal_solve (public API) for a config, best of 3 after a warm-up."""
import os, sys, time
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2510_11023_b200 as pfb
cfg = int(sys.argv[1])
c = pfb.problems.CONFIGS[cfg]
P = int(sys.argv[2]) if len(sys.argv) > 2 else c["nt"]
prob = pfb.config_problem(cfg); op = pfb.build_sine_operator(c["modes"], dims=c["dims"])
g = pfb.TimeGrids(c["t_final"], P, c["m"])
pfb.parareal_solve(prob, op, g, tol=c["tol"], k_max=P + 1)
best = 1e9
for _ in range(3):
    t0 = time.perf_counter()
    it, rep = pfb.parareal_solve(prob, op, g, tol=c["tol"], k_max=P + 1)
    best = min(best, time.perf_counter() - t0)
print(f"config {cfg} P={P} PF_PIPELINE={os.environ.get('PF_PIPELINE', 'default')}: time-to-tol {best:.4f} s, "
      f"{rep.iterations} iterations, final diff {rep.diffs[-1]:.3e}")
