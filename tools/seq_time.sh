# run_fine_sequential at config 3 full size (N = 65536): device time and PCG iterations
python - <<'PY'
import sys, time, numpy as np
sys.path.insert(0, ".")
import paper_2510_11023_b200 as pfb
from paper_2510_11023_b200 import _lib
prob = pfb.config_problem(3); op = pfb.build_sine_operator(512); g = pfb.TimeGrids(2.0, 64, 1024)
pfb.run_fine_sequential(prob, op, g)
ctx = _lib.context_for(prob, op, g); _lib.lib.pf_reset_stats(ctx.handle)
st, secs = pfb.run_fine_sequential(prob, op, g)
s = ctx.stats()
print(f"run_fine_sequential config 3: {secs:.3f} s wall, kernel {s['last_fine_ms']:.1f} ms, PCG it/solve {s['pcg_iterations']/max(s['solves'],1):.4f}")
PY
