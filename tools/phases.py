"""Per-phase cycle breakdown of slice 0 of the config-3 fine sweep (needs a -DPF_PHASE_TIMING build)."""
import ctypes as C, sys, numpy as np
sys.path.insert(0, "/root/repo")
import paper_2510_11023_b200 as pfb
from paper_2510_11023_b200 import _lib
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
c = pfb.problems.CONFIGS[cfg]
prob = pfb.config_problem(cfg); op = pfb.build_sine_operator(c["modes"]); g = pfb.TimeGrids(c["t_final"], c["nt"], c["m"])
tr = pfb.run_coarse(prob, op, g)
pfb.fine_sweep_intervals(tr, 0, c["nt"], op, g, prob)
buf = (C.c_longlong * 16)()
_lib.lib.pf_debug_phases(buf, 1)
pfb.fine_sweep_intervals(tr, 0, c["nt"], op, g, prob)
_lib.lib.pf_debug_phases(buf, 0)
names = {0: "from step entry (misc)", 1: "synth FFT", 2: "pointwise (fused)", 3: "analysis FFT", 4: "residual+reduce",
         5: "CG apply_k (2 FFT)", 6: "CG update+reduce", 7: "finite check", 8: "block start (helper wait)",
         9: "near hist + extrap", 10: "path write/loop", 11: "HELPER wait for progress",
         12: "HELPER far GEMM", 13: "HELPER bracket", 14: "HELPER publish+loop"}
tot = sum(buf)
for k in range(16):
    if buf[k]:
        print(f"{names.get(k, k):28s} {buf[k]/c['m']:10.0f} cyc/substep  {100*buf[k]/tot:5.1f}%")
print("total cycles/substep", tot / c["m"], " stats", _lib.context_for(prob, op, g).stats())
