"""Ad-hoc 2-D GPU vs oracle check (dev tool)."""
import sys, time, numpy as np
sys.path.insert(0, "/root/repo")
import paper_2510_11023_b200 as pfb
import oracle
from oracle import problems as OP
def rel(a, b): return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
for cfg, M, nt, m in [(4, 8, 4, 8), (4, 16, 6, 16), (5, 16, 4, 8), (4, 32, 8, 16)]:
    prob = pfb.config_problem(cfg, modes=M); op = pfb.build_sine_operator(M, dims=2)
    g = pfb.TimeGrids(1.0, nt, m); og = oracle.TimeGrids(1.0, nt, m)
    osp = oracle.Sine2D(M, pcg_tol=op.pcg_tol)
    oprob = OP.config(cfg, modes=M)
    t0 = time.time(); tr = pfb.run_coarse(prob, op, g); t1 = time.time()
    otr = oracle.run_coarse(oprob, osp, og)
    print(f"cfg{cfg} M{M}: run_coarse err {rel(tr, otr):.2e} ({(t1-t0)*1e3:.0f} ms)")
    fs = pfb.fine_sweep_intervals(otr, 0, nt, op, g, prob)
    ofs = oracle.fine_sweep_intervals(otr, 0, nt, osp, og, oprob)
    print(f"   fine sweep err {rel(fs, ofs):.2e}")
    t0 = time.time(); it, rep = pfb.parareal_solve(prob, op, g, tol=1e-12, k_max=nt + 1); t1 = time.time()
    oit, orep = oracle.parareal_solve(oprob, osp, og, tol=1e-12, k_max=nt + 1)
    print(f"   parareal err {rel(it.states, oit.states):.2e} iters {rep.iterations} vs {orep.iterations} ({(t1-t0)*1e3:.0f} ms) "
          f"pcg/solve {rep.device_stats['pcg_iterations']/max(rep.device_stats['solves'],1):.2f}")
# full-size cfg4 single sweep timing
for cfg in (4,):
    c = pfb.problems.CONFIGS[cfg]
    prob = pfb.config_problem(cfg); op = pfb.build_sine_operator(c["modes"], dims=2)
    g = pfb.TimeGrids(1.0, c["nt"], c["m"])
    U = np.tile(pfb.initial_state(prob, op), (c["nt"] + 1, 1))
    t0 = time.time(); fs = pfb.fine_sweep_intervals(U, 0, c["nt"], op, g, prob); t1 = time.time()
    ctx = pfb._lib.context_for(prob, op, g)
    print(f"cfg{cfg} full fine sweep (uniform start): {t1-t0:.2f} s, stats {ctx.stats()}")
