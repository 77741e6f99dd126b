"""Determinism and cross-engine agreement of the config-3-shaped sweep (M = 512): repeated runs
bitwise, helper vs inline bitwise, DMMA vs DFMA far history to rounding.  One process per setting."""
import os, subprocess, sys, tempfile
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
CODE = """
import sys, numpy as np
sys.path.insert(0, {root!r})
import paper_2510_11023_b200 as p
pr = p.config_problem(3); op = p.build_sine_operator(512)
g = p.TimeGrids(2.0, 16, 96)
t = p.run_coarse(pr, op, g)
outs = [p.fine_sweep_intervals(t, 0, 16, op, g, pr) for _ in range(3)]
np.savez(sys.argv[1], a=outs[0], b=outs[1], c=outs[2])
"""
def run(env):
    with tempfile.TemporaryDirectory() as d:
        f = os.path.join(d, "o.npz")
        subprocess.run([sys.executable, "-c", CODE.format(root=ROOT), f], check=True, env=dict(os.environ, **env))
        z = np.load(f)
        return [z[k] for k in "abc"]
res = {}
for name, env in {"dfma helper": {}, "dfma inline": {"PF_NO_HELPERS": "1"}, "dmma helper": {"PF_FAR_TC": "1"},
                  "dmma inline": {"PF_NO_HELPERS": "1", "PF_FAR_TC": "1"}, "tma helper": {"PF_FAR_TC": "2"}}.items():
    r = run(env)
    res[name] = r[0]
    print(f"{name:12s} repeat bitwise: {np.array_equal(r[0], r[1]) and np.array_equal(r[1], r[2])}")
ref = res["dfma inline"]
for k, v in res.items():
    print(f"{k:12s} vs dfma inline: rel {np.linalg.norm(v - ref) / np.linalg.norm(ref):.3e}  bitwise {np.array_equal(v, ref)}")
print("dmma helper vs dmma inline bitwise:", np.array_equal(res["dmma helper"], res["dmma inline"]),
      " tma vs dmma inline:", np.array_equal(res["tma helper"], res["dmma inline"]))
