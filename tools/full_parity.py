"""Config 3 at full size on device vs the full-size CPU oracle fixture (tests/golden/oracle_cfg3_full.npz)."""
import os, sys, numpy as np
sys.path.insert(0, "/root/repo")
import paper_2510_11023_b200 as pfb
want = np.load("/root/repo/tests/golden/oracle_cfg3_full.npz")
prob = pfb.config_problem(3); op = pfb.build_sine_operator(512); g = pfb.TimeGrids(2.0, 64, 1024)
it, rep = pfb.parareal_solve(prob, op, g, tol=1e-12, k_max=65)
rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
print(f"iterations device {rep.iterations} oracle {int(want['iterations'])}")
print(f"states rel L2 {rel(it.states, want['states']):.3e}, fine endpoints rel L2 {rel(it.fine_endpoints, want['fine_endpoints']):.3e}")
print("diffs device", np.array(rep.diffs)); print("diffs oracle", want["diffs"])
