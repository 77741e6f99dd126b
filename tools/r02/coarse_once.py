"""One 2-D run_coarse (config 4 shape, P from argv) for kernel launch lists."""
import sys
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2510_11023_b200 as pfb
P = int(sys.argv[1]) if len(sys.argv) > 1 else 16
c = pfb.problems.CONFIGS[4]
prob = pfb.config_problem(4); op = pfb.build_sine_operator(128, dims=2)
g = pfb.TimeGrids(1.0, P, c["m"])
pfb.run_coarse(prob, op, g)
print("ok")
