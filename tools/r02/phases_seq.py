"""Phase breakdown of the config-3 sequential solver (run_fine_sequential: slice 0
over nt*m substeps, far history split-K over the helper CTAs) with the
-DPF_PHASE_TIMING library (tools/phases.sh PHASE_SO=phase ...)."""
import ctypes as C, sys, time
sys.path.insert(0, "/root/repo")
import paper_2510_11023_b200 as pfb
from paper_2510_11023_b200 import _lib
nt = int(sys.argv[1]) if len(sys.argv) > 1 else 64
c = pfb.problems.CONFIGS[3]
prob = pfb.config_problem(3); op = pfb.build_sine_operator(512); g = pfb.TimeGrids(c["t_final"] * nt / 64, nt, c["m"])
buf = (C.c_longlong * 16)()
pfb.run_fine_sequential(prob, op, g)
_lib.lib.pf_debug_phases(buf, 1)
t0 = time.perf_counter(); pfb.run_fine_sequential(prob, op, g); t1 = time.perf_counter()
_lib.lib.pf_debug_phases(buf, 0)
N = nt * c["m"]
names = {0: "from step entry", 1: "synth FFT", 2: "pointwise", 3: "analysis FFT", 4: "residual+reduce",
         5: "CG apply_k", 6: "CG update+reduce", 7: "finite check", 8: "block start (helper wait)",
         9: "near hist + extrap", 10: "path write/loop", 11: "HELPER wait for progress",
         12: "HELPER far GEMM", 13: "HELPER bracket", 14: "HELPER publish+loop"}
tot = sum(buf)
print(f"run_fine_sequential N={N}: {t1 - t0:.3f} s")
for k in range(16):
    if buf[k]:
        print(f"{names.get(k, k):28s} {buf[k]/N:10.0f} cyc/substep  {100*buf[k]/tot:5.1f}%")
st = _lib.context_for(prob, op, g).stats()
print("pcg iterations per solve", st["pcg_iterations"] / max(st["solves"], 1), st)
