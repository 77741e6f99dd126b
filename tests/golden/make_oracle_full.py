"""Full-size oracle runs of the BASELINE configs (CPU, long): fixtures for the
device parity tests at full size.

    python tests/golden/make_oracle_full.py 3      # config 3: ~2 h on 8 cores
    python tests/golden/make_oracle_full.py 4 2    # config 4, first 2 iterations (2-D, oracle.Sine2D)

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


def main(i, k_max=None):
    M, nt, m, alpha, T, tol = P.CONFIG_GRIDS[i]
    prob = P.config(i)
    space = oracle.Sine1D(M) if i <= 3 else oracle.Sine2D(M, pcg_tol=1e-13)
    grids = oracle.TimeGrids(T, nt, m)
    t0 = time.time()
    it, rep = oracle.parareal_solve(prob, space, grids, tol=tol, k_max=k_max or nt + 1)
    path = os.path.join(HERE, f"oracle_cfg{i}_full.npz" if k_max is None else f"oracle_cfg{i}_full_k{k_max}.npz")
    np.savez_compressed(path, states=it.states, fine_endpoints=it.fine_endpoints, diffs=np.array(rep.diffs),
                        iterations=np.array(rep.iterations))
    print(f"config {i}: {rep.iterations} iterations, diffs {rep.diffs}, {time.time() - t0:.0f} s -> {path}")


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 3, int(sys.argv[2]) if len(sys.argv) > 2 else None)
