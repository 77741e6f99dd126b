"""Per-iteration phase times of the parareal driver on one GPU (DeviceOps state
machine, no torch.distributed): fine sweep vs correction sweep, PCG counters.
    python tools/r02/phase_times.py CONFIG [P]"""
import sys
import time

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
import torch
import paper_2510_11023_b200 as pfb
from paper_2510_11023_b200.parallel import DeviceOps

cfg = int(sys.argv[1])
c = pfb.problems.CONFIGS[cfg]
P = int(sys.argv[2]) if len(sys.argv) > 2 else c["nt"]
prob = pfb.config_problem(cfg)
op = pfb.build_sine_operator(c["modes"], dims=c["dims"])
g = pfb.TimeGrids(c["t_final"], P, c["m"])
ops = DeviceOps(prob, op, g, 0)
with ops.scope():
    fold = ops.empty(P)
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ops.init()
        torch.cuda.synchronize()
        tinit = time.perf_counter() - t0
        rows = []
        for k in range(P + 1):
            lo = 0 if k == 0 else ops.frozen()
            s0 = ops.ctx.stats()
            ta = time.perf_counter()
            if lo < P:
                ops.fine(lo, P, fold[lo:])
            torch.cuda.synchronize()
            tb = time.perf_counter()
            s1 = ops.ctx.stats()
            diff = ops.correct(fold, k)
            torch.cuda.synchronize()
            tc = time.perf_counter()
            s2 = ops.ctx.stats()
            rows.append((k, lo, 1e3 * (tb - ta), 1e3 * (tc - tb), diff,
                         (s1["pcg_iterations"] - s0["pcg_iterations"]) / max(1, s1["solves"] - s0["solves"]),
                         (s2["pcg_iterations"] - s1["pcg_iterations"]) / max(1, s2["solves"] - s1["solves"]),
                         s2["kernel_launches"] - s1["kernel_launches"]))
            if diff < c["tol"]:
                break
        total = time.perf_counter() - t0
    print(f"config {cfg} P={P}: init (run_coarse) {1e3*tinit:.1f} ms, total {total:.3f} s, {len(rows)} iterations")
    print(" k  lo   fine_ms  corr_ms      diff   pcg/solve(fine) pcg/solve(corr) corr_launches")
    for r in rows:
        print(f"{r[0]:2d} {r[1]:3d} {r[2]:9.2f} {r[3]:8.2f} {r[4]:9.2e} {r[5]:8.2f} {r[6]:8.2f} {r[7]:8d}")
    print(f"sum fine {sum(r[2] for r in rows):.1f} ms, sum corr {sum(r[3] for r in rows):.1f} ms")
