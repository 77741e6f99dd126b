"""Ad-hoc GPU parity sweep (dev tool): prints max errors vs the oracle."""
import sys, time, numpy as np
sys.path.insert(0, "/root/repo")
import paper_2510_11023_b200 as pfb
import oracle

def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))

# --- Chebyshev bridge vs oracle (== reference bitwise) ---
p42 = pfb.get_problem("paper42")
for deg, nt, m in [(8, 8, 4), (16, 16, 4), (33, 8, 64)]:
    cop = pfb.build_operator(deg, 0.0, 1.0); oop = oracle.build_operator(deg, 0.0, 1.0)
    g = pfb.TimeGrids(1.0, nt, m); og = oracle.TimeGrids(1.0, nt, m)
    t0 = time.time(); tr = pfb.run_coarse(p42, cop, g); t1 = time.time()
    otr = oracle.run_coarse(p42, oop, og)
    print(f"cheb deg{deg} run_coarse err {rel(tr, otr):.2e} ({(t1-t0)*1e3:.1f} ms)")
    fs = pfb.fine_sweep_intervals(otr, 0, nt, cop, g, p42)
    ofs = oracle.fine_sweep_intervals(otr, 0, nt, oop, og, p42)
    print(f"cheb deg{deg} fine_sweep err {rel(fs, ofs):.2e}")
    it, rep = pfb.parareal_solve(p42, cop, g, tol=1e-12, k_max=nt + 1)
    oit, orep = oracle.parareal_solve(p42, oop, og, tol=1e-12, k_max=nt + 1)
    print(f"cheb deg{deg} parareal err {rel(it.states, oit.states):.2e} iters {rep.iterations} vs {orep.iterations}; diffs {rep.diffs[:3]} vs {orep.diffs[:3]}")
# --- sine 1-D vs oracle ---
for cfg, M, nt, m in [(1, 32, 8, 64), (2, 64, 16, 256), (3, 64, 8, 64)]:
    prob = pfb.config_problem(cfg, modes=M); op = pfb.build_sine_operator(M)
    g = pfb.TimeGrids(prob.t_final, nt, m); og = oracle.TimeGrids(prob.t_final, nt, m)
    osp = oracle.Sine1D(M)
    tr = pfb.run_coarse(prob, op, g); otr = oracle.run_coarse(prob, osp, og)
    print(f"sine cfg{cfg} M{M} run_coarse err {rel(tr, otr):.2e}")
    fs = pfb.fine_sweep_intervals(otr, 0, nt, op, g, prob)
    ofs = oracle.fine_sweep_intervals(otr, 0, nt, osp, og, prob)
    print(f"sine cfg{cfg} M{M} fine_sweep err {rel(fs, ofs):.2e}")
    t0 = time.time(); it, rep = pfb.parareal_solve(prob, op, g, tol=1e-12, k_max=nt + 1); t1 = time.time()
    oit, orep = oracle.parareal_solve(prob, osp, og, tol=1e-12, k_max=nt + 1)
    print(f"sine cfg{cfg} parareal err {rel(it.states, oit.states):.2e} iters {rep.iterations} vs {orep.iterations} ({(t1-t0)*1e3:.1f} ms) stats {rep.device_stats}")
    print("   diffs gpu ", ["%.2e" % d for d in rep.diffs])
    print("   diffs orc ", ["%.2e" % d for d in orep.diffs])
# --- full-size cfg3 fine sweep timing ---
prob = pfb.config_problem(3); op = pfb.build_sine_operator(512)
g = pfb.TimeGrids(2.0, 64, 1024)
tr = pfb.run_coarse(prob, op, g)
for rep_ in range(2):
    t0 = time.time(); fs = pfb.fine_sweep_intervals(tr, 0, 64, op, g, prob); t1 = time.time()
    ctx = pfb._lib.context_for(prob, op, g)
    print(f"cfg3 fine sweep: {(t1-t0)*1e3:.1f} ms wall, stats {ctx.stats()}")
