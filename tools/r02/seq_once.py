"""One config-3 run_fine_sequential (N = 65 536 substeps) for an ncu capture."""
import sys, time
sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import paper_2510_11023_b200 as pfb
pr = pfb.config_problem(3); op = pfb.build_sine_operator(512); g = pfb.TimeGrids(2.0, 64, 1024)
t = time.perf_counter(); s, sec = pfb.run_fine_sequential(pr, op, g); print("seq s", time.perf_counter() - t)
