"""run_fine_sequential on device: parity at reduced size, timing at config-3 size."""
import sys, time, numpy as np
sys.path.insert(0, "/root/repo")
import paper_2510_11023_b200 as pfb
import oracle
from oracle import problems as OP
def rel(a, b): return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
for cfg, M, nt, m in [(1, 32, 8, 64), (3, 64, 8, 128), (2, 64, 16, 256)]:
    prob = pfb.config_problem(cfg, modes=M); op = pfb.build_sine_operator(M)
    c = pfb.problems.CONFIGS[cfg]
    g = pfb.TimeGrids(c["t_final"], nt, m)
    t0 = time.time(); s, _ = pfb.run_fine_sequential(prob, op, g); t1 = time.time()
    os_, _ = oracle.run_fine_sequential(OP.config(cfg, modes=M), oracle.Sine1D(M), oracle.TimeGrids(c["t_final"], nt, m))
    st = pfb._lib.context_for(prob, op, g).stats()
    print(f"cfg{cfg} M{M} N={nt*m}: seq err {rel(s, os_):.2e} ({(t1-t0)*1e3:.0f} ms, helpers used: {st['helper_launches']})")
    if cfg == 2:  # alpha = 1: the full-history solver equals the parareal fixed point
        ch = pfb.chain_fine(prob, op, g)
        print(f"   alpha=1: |seq - chain_fine| rel {rel(s, ch):.2e}")
prob = pfb.config_problem(3); op = pfb.build_sine_operator(512); g = pfb.TimeGrids(2.0, 64, 1024)
for rep in range(2):
    t0 = time.time(); s, secs = pfb.run_fine_sequential(prob, op, g); t1 = time.time()
    st = pfb._lib.context_for(prob, op, g).stats()
    print(f"cfg3 full run_fine_sequential (N=65536): {t1-t0:.2f} s wall, kernel {st['last_fine_ms']:.0f} ms, pcg/solve {st['pcg_iterations']/max(st['solves'],1):.2f}")
it, rep_ = pfb.parareal_solve(prob, op, g, tol=1e-12, k_max=65, reference=s)
print("parareal vs full-history solver at T:", rep_.errors_vs_reference[-1], "(SURVEY: parareal converges to chain_fine, not to the full-history solution)")
