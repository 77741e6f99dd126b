"""Edge sizes of the 1-D sweep against the oracle: other mode counts (M = 1024, 256, 128: the engines without
side warps / grouped helper) and, at M = 512 (side warps + grouped TMA-fed DMMA helper), substep counts that are
not multiples of the block (8) or super-block (32) lengths, with and without helper CTAs."""
import os, subprocess, sys
import numpy as np
sys.path.insert(0, "/root/repo")
if len(sys.argv) > 1 and sys.argv[1] == "child":
    import paper_2510_11023_b200 as pfb, oracle
    M, nt, m = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
    T = 2.0 * nt * m / 65536
    prob = pfb.config_problem(3, modes=M); op = pfb.build_sine_operator(M); g = pfb.TimeGrids(T, nt, m)
    tr = pfb.run_coarse(prob, op, g)
    got = pfb.fine_sweep_intervals(tr, 0, nt, op, g, prob)
    osp = oracle.Sine1D(M); og = oracle.TimeGrids(T, nt, m); op3 = oracle.problems.config(3, modes=M)
    otr = oracle.run_coarse(op3, osp, og)
    want = oracle.fine_sweep_intervals(otr, 0, nt, osp, og, op3)
    print(f"M={M:5d} nt={nt} m={m:4d} {os.environ.get('PF_NO_HELPERS', '0')}: coarse {np.linalg.norm(tr - otr) / np.linalg.norm(otr):.2e} "
          f"sweep {np.linalg.norm(got - want) / np.linalg.norm(want):.2e}")
    sys.exit(0)
cases = [(1024, 4, 24), (256, 4, 24), (128, 4, 24), (512, 3, 1), (512, 3, 7), (512, 3, 8), (512, 3, 9), (512, 3, 33),
         (512, 3, 40), (512, 2, 100), (512, 2, 129)]
for M, nt, m in cases:
    for nh in ("0", "1") if M == 512 else ("0",):
        subprocess.run([sys.executable, __file__, "child", str(M), str(nt), str(m)], env=dict(os.environ, PF_NO_HELPERS=nh))
