"""Substep durations of the traced slice's early phase (needs a -DPF_TRACE build with -DPF_TRACE_SLICE=n):
duration ~ setup pair (~8.9k cycles) + PCG iterations x ~4.9k."""
import ctypes as C, sys, numpy as np
sys.path.insert(0, "/root/repo")
import paper_2510_11023_b200 as pfb
from paper_2510_11023_b200 import _lib
c = pfb.problems.CONFIGS[3]
prob = pfb.config_problem(3); op = pfb.build_sine_operator(c["modes"]); g = pfb.TimeGrids(c["t_final"], c["nt"], c["m"])
tr = pfb.run_coarse(prob, op, g)
pfb.fine_sweep_intervals(tr, 0, c["nt"], op, g, prob)
pfb.fine_sweep_intervals(tr, 0, c["nt"], op, g, prob)
m = c["m"]
lt = (C.c_longlong * (m + 1))()
_lib.lib.pf_debug_looptop(lt, m + 1)
d = np.diff(np.array(lt[1:m + 1], dtype=np.int64)).astype(float)
base = np.median(d[600:900])
print("steady substep", base)
print("r=1..32 (est. extra PCG iterations):", " ".join(f"{(v - base) / 4900:.1f}" for v in d[:32]))
for w0 in range(32, 320, 16):
    seg = d[w0:w0 + 16]
    print(f"r {w0 + 1:4d}..{w0 + 16:4d}: mean {seg.mean():8.0f}  extra iterations ~{(seg.mean() - base) / 4900:.2f}")
print("early-phase overhead (cycles above steady, r <= 320):", (d[:320] - base).sum(), "=", (d[:320] - base).sum() / 1.965e6, "ms")
