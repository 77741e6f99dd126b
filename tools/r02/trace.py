"""Per-warp timeline of 8 substeps of one slice CTA of the config-3 sweep (needs a -DPF_TRACE build:
tools/r02/trace.sh).  For every trace point: cycles since the substep's loop top, averaged over the
traced substeps, for the earliest and the latest warp, and the increment of the latest warp."""
import ctypes as C, sys, numpy as np
sys.path.insert(0, "/root/repo")
import paper_2510_11023_b200 as pfb
from paper_2510_11023_b200 import _lib
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
c = pfb.problems.CONFIGS[cfg]
prob = pfb.config_problem(cfg); op = pfb.build_sine_operator(c["modes"]); g = pfb.TimeGrids(c["t_final"], c["nt"], c["m"])
tr = pfb.run_coarse(prob, op, g)
pfb.fine_sweep_intervals(tr, 0, c["nt"], op, g, prob)
pfb.fine_sweep_intervals(tr, 0, c["nt"], op, g, prob)
buf = (C.c_longlong * 4096)()
_lib.lib.pf_debug_trace(buf)
t = np.array(buf[:], dtype=np.int64).reshape(8, 8, 64)   # [warp][substep][point]
names = {0: "loop top", 1: "block start done", 2: "near hist + guess done", 3: "synth input + bar",
         4: "inv r8 #1", 5: "inv r8 #2", 6: "inv r4", 7: "last inv + pointwise + first fwd + bar",
         8: "fwd r4", 9: "fwd r8 #1", 10: "fwd r8 #2", 11: "gather + residual (before sum4)", 12: "sum4 done",
         13: "pinv, z, p done", 46: "step end", 47: "path/ring write done"}
for it in (1, 2):
    b = 14 + (it - 1) * 16
    names.update({b: f"cg{it} synth input + bar", b + 1: f"cg{it} inv r8 #1", b + 2: f"cg{it} inv r8 #2", b + 3: f"cg{it} inv r4",
                  b + 4: f"cg{it} last inv * d + first fwd + bar", b + 5: f"cg{it} fwd r4", b + 6: f"cg{it} fwd r8 #1",
                  b + 7: f"cg{it} fwd r8 #2", b + 8: f"cg{it} gather + pq (before sum2)", b + 9: f"cg{it} sum2 done",
                  b + 10: f"cg{it} update (before sum2)", b + 11: f"cg{it} sum2 done"})
order = [0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13] + list(range(14, 26)) + list(range(30, 42)) + [46, 47]
t0 = t[:, :, 0].min(axis=0)                               # substep start: earliest warp at loop top
steps = [s for s in range(8) if t0[s] > 0]
print(f"config {cfg}: traced substeps {len(steps)}; cycles since loop top (mean over substeps)")
print(f"{'point':44s} {'first warp':>10s} {'last warp':>10s} {'+last':>7s}   n")
prev = 0.0
for p in order:
    ok = [s for s in steps if (t[:, s, p] > 0).all() and (t[:, s, p] >= t0[s]).all()]
    if not ok:
        continue
    rel = np.array([[t[w, s, p] - t0[s] for w in range(8)] for s in ok], dtype=float)
    lo, hi = rel.min(axis=1).mean(), rel.max(axis=1).mean()
    print(f"{names.get(p, p):44s} {lo:10.0f} {hi:10.0f} {hi - prev:7.0f}   {len(ok)}")
    prev = hi
nxt = [t[:, s + 1, 0].min() - t0[s] for s in steps if s + 1 in steps]
print("substep length (loop top to loop top):", np.mean(nxt) if nxt else None)
for s in steps:
    print("substep", s, "block-start" if (s % 8) == ((513 - 1) % 8) else "", "length", (t[:, s + 1, 0].min() - t0[s]) if s + 1 in steps else None)

# substep durations over the whole sweep (loop top to loop top), in windows of 64 substeps
m = c["m"]
lt = (C.c_longlong * (m + 1))()
_lib.lib.pf_debug_looptop(lt, m + 1)
lt = np.array(lt[:], dtype=np.int64)
d = np.diff(lt[1:m + 1]).astype(float)
print("substep duration by window of 64 substeps (mean cycles; block-start substeps' mean; max):")
for w0 in range(0, m - 1, 64):
    seg = d[w0:w0 + 64]
    idx = np.arange(w0 + 1, w0 + 1 + len(seg))
    bs = seg[(idx - 1) % 8 == 0]
    print(f"  r {w0 + 1:5d}..{w0 + len(seg):5d}: mean {seg.mean():8.0f}  block-start mean {bs.mean() if len(bs) else 0:8.0f}  max {seg.max():8.0f}")
print("total cycles", lt[m] - lt[1], "=", (lt[m] - lt[1]) / 1.965e6, "ms at 1965 MHz")
# per-warp arrival (cycles since loop top, mean over the traced substeps) at the setup transform's points
print("per-warp arrival times (warp 0..7):")
for p in (3, 4, 5, 6, 7, 8, 9, 10, 14, 15, 16):
    ok = [s for s in steps if (t[:, s, p] > 0).all()]
    if ok:
        rel = np.array([[t[w, s, p] - t0[s] for w in range(8)] for s in ok], dtype=float).mean(axis=0)
        print(f"  {names.get(p, p):40s} " + " ".join(f"{v:6.0f}" for v in rel))
