import sys, time
sys.path.insert(0, "/root/repo")
import paper_2510_11023_b200 as pfb
c = pfb.problems.CONFIGS[4]
prob = pfb.config_problem(4); op = pfb.build_sine_operator(128, dims=2)
g = pfb.TimeGrids(c["t_final"], int(sys.argv[1]), c["m"])
pfb.run_coarse(prob, op, g)
t0 = time.perf_counter(); pfb.run_coarse(prob, op, g); t1 = time.perf_counter()
print(f"run_coarse nt={g.nt}: {1e3*(t1-t0):.2f} ms, {1e3*(t1-t0)/g.nt:.3f} ms/step")
