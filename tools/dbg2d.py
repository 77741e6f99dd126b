import sys, numpy as np
sys.path.insert(0, "/root/repo")
import paper_2510_11023_b200 as pfb
import oracle
from oracle import problems as OP
def rel(a, b): return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
for M, nt in [(16, 6), (32, 4), (64, 2), (128, 2)]:
    prob = pfb.config_problem(4, modes=M); op = pfb.build_sine_operator(M, dims=2)
    g = pfb.TimeGrids(1.0, nt, 4); og = oracle.TimeGrids(1.0, nt, 4)
    osp = oracle.Sine2D(M); oprob = OP.config(4, modes=M)
    otr = oracle.run_coarse(oprob, osp, og)
    for n in range(nt):
        try:
            got = pfb.coarse_step(otr[: n + 1], op, g, prob)
            print(f"M{M} coarse n={n}: err {rel(got, otr[n+1]):.2e}", pfb._lib.context_for(prob, op, g).stats()["pcg_iterations"])
        except Exception as e:
            print(f"M{M} coarse n={n}: {type(e).__name__} {e}")
