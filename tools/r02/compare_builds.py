"""Bitwise comparison of the M = 512 sweep between library builds (refactors that must not change arithmetic):
    python tools/r02/compare_builds.py tools/variants/a.so tools/variants/b.so ..."""
import os, subprocess, sys, tempfile
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
CODE = """
import sys, numpy as np
sys.path.insert(0, {root!r})
import paper_2510_11023_b200 as p
pr = p.config_problem(3); op = p.build_sine_operator(512)
g = p.TimeGrids(2.0 * 6 * 200 / 65536, 6, 200)
t = p.run_coarse(pr, op, g)
np.save(sys.argv[1], p.fine_sweep_intervals(t, 0, 6, op, g, pr))
"""
outs = []
for lib in sys.argv[1:]:
    with tempfile.TemporaryDirectory() as d:
        f = os.path.join(d, "o.npy")
        subprocess.run([sys.executable, "-c", CODE.format(root=ROOT), f], check=True,
                       env=dict(os.environ, PARAFRAC_B200_LIB=os.path.abspath(lib)))
        outs.append(np.load(f))
for lib, o in zip(sys.argv[1:], outs):
    print(f"{lib}: bitwise equal to the first: {np.array_equal(o, outs[0])}  rel {np.linalg.norm(o - outs[0]) / np.linalg.norm(outs[0]):.2e}")
