"""Full-size oracle runs of the BASELINE configs (CPU, long): fixtures for the
device parity tests at full size.

    python tests/golden/make_oracle_full.py 3      # config 3: ~1 h on 8 cores

Writes tests/golden/oracle_cfg<i>_full.npz with the parareal iterate (states),
the diff sequence and the iteration count of the oracle restatement
(oracle/, sine spectral Galerkin with dense assembly + LAPACK solves).
"""

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402
from oracle import problems as P  # noqa: E402


def main(i):
    M, nt, m, alpha, T, tol = P.CONFIG_GRIDS[i]
    prob = P.config(i)
    space = oracle.Sine1D(M)
    grids = oracle.TimeGrids(T, nt, m)
    t0 = time.time()
    it, rep = oracle.parareal_solve(prob, space, grids, tol=tol, k_max=nt + 1)
    path = os.path.join(HERE, f"oracle_cfg{i}_full.npz")
    np.savez_compressed(path, states=it.states, fine_endpoints=it.fine_endpoints, diffs=np.array(rep.diffs),
                        iterations=np.array(rep.iterations))
    print(f"config {i}: {rep.iterations} iterations, diffs {rep.diffs}, {time.time() - t0:.0f} s -> {path}")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 3)
