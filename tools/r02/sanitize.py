"""Small config-3-shaped sweeps for compute-sanitizer (one tool per gpurun call):
M = 512 (the Q = 1024 radix-8 engine), 8 slices + 8 helper CTAs (cooperative
launch, release/acquire block flags), m = 40 substeps (5 history blocks), the
head-start launch of slice 0 is off (below its size threshold), plus one
parareal solve (k_coarse correction sweeps, frozen prefix), the split-K
sequential solver and a 2-D config-4-shaped sweep."""
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import numpy as np
import paper_2510_11023_b200 as pfb
from paper_2510_11023_b200 import _lib

prob = pfb.config_problem(3)
op = pfb.build_sine_operator(512)
g = pfb.TimeGrids(2.0, 8, 40)
traj = pfb.run_coarse(prob, op, g)
out = pfb.fine_sweep_intervals(traj, 0, 8, op, g, prob)
ctx = _lib.context_for(prob, op, g)
assert ctx.stats()["helper_launches"] >= 1
it, rep = pfb.parareal_solve(prob, op, g, tol=1e-12, k_max=9)
seq, _ = pfb.run_fine_sequential(prob, op, pfb.TimeGrids(2.0, 4, 64))
p4 = pfb.config_problem(4, modes=32)
op4 = pfb.build_sine_operator(32, dims=2)
g4 = pfb.TimeGrids(1.0, 4, 9)
t4 = pfb.run_coarse(p4, op4, g4)
o4 = pfb.fine_sweep_intervals(t4, 0, 4, op4, g4, p4)
print("sanitize workload ok:", float(np.abs(out).max()), rep.iterations, float(np.abs(seq).max()), float(np.abs(o4).max()))
