"""Which slice finishes last in a full config-3 sweep (all 64 slices together)?
Prints per-slice finish times relative to the earliest finisher (GPU globaltimer)."""
import ctypes as C, sys, numpy as np
sys.path.insert(0, "/root/repo")
import paper_2510_11023_b200 as pfb
from paper_2510_11023_b200 import _lib
prob = pfb.config_problem(3); op = pfb.build_sine_operator(512); g = pfb.TimeGrids(2.0, 64, 1024)
tr = pfb.run_coarse(prob, op, g)
ctx = _lib.context_for(prob, op, g)
acc = np.zeros(64)
st = np.zeros(64)
for rep in range(6):
    pfb.fine_sweep_intervals(tr, 0, 64, op, g, prob)
    buf = (C.c_longlong * 128)()
    ctx.check(_lib.lib.pf_debug_slice_times_ns(ctx.handle, buf, 64))
    t = np.array(buf[:], dtype=float).reshape(64, 2)
    if rep:
        acc += (t[:, 1] - t[:, 1].min()) / 1e3
        st += (t[:, 0] - t[:, 0].min()) / 1e3
acc /= 5
st /= 5
order = np.argsort(-acc)
print("sweep ms", ctx.stats()["last_fine_ms"])
print("latest finishers (us after the first):", [(int(i), round(acc[i], 1)) for i in order[:10]])
print("earliest:", [(int(i), round(acc[i], 1)) for i in order[-5:]])
print("per slice:", " ".join(f"{v:.0f}" for v in acc))
print("entry offsets (us):", " ".join(f"{v:.0f}" for v in st))
