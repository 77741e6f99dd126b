"""Initial guesses of the parareal correction sweep's coarse solves (2-D, config 4
space, reduced P): PCG iterations per solve with
  drift : G_old[n] + (U_next[n] - U_cur[n])          (round 1 device rule)
  pdrift: G_old[n] + Pinv (sum_j w_j (U_next[j] - U_cur[j]))   (the history
          change pushed through the preconditioner, Pinv ~ A^-1)
on the oracle's exact coarse steps (oracle.Sine2D, PCG tol 1e-13)."""
import math
import os
import sys

os.environ.setdefault("OPENBLAS_NUM_THREADS", "8")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np

import oracle
from oracle import problems as P
from oracle import stepping as S
from oracle.spaces import pcg
from oracle.weights import gamma_2_minus, history_weights, weights_for

cfg, nt, m = 4, int(sys.argv[1]) if len(sys.argv) > 1 else 16, 16
M = 128
prob = P.config(cfg)
sp = oracle.Sine2D(M, pcg_tol=1e-13)
g = oracle.TimeGrids(1.0, nt, m)
alpha = prob.alpha
gam = g.dT ** alpha * gamma_2_minus(alpha)
U = S.run_coarse(prob, sp, g)
# one parareal iteration with the oracle to get U_next, G_old
fold = S.fine_sweep_intervals(U, 0, nt, sp, g, prob)
gold = U[1:].copy()
Un = np.empty_like(U)
Un[0] = U[0]
its = {"drift": [], "pdrift": [], "prev": []}
for n in range(nt):
    H = Un[: n + 1]
    b = weights_for(alpha).on_grid(1, n + 2)
    w = history_weights(b, n)
    d = sp.operator(H[n], n * g.dT, prob, batched=False)
    rhs = w @ H + gam * sp.source(H[n], n * g.dT, prob, batched=False)
    dbar = float(np.sum(d))
    pinv = (1.0 / (1.0 + gam * dbar * math.pi ** 2 * sp.k2)).reshape(-1)
    A = lambda v: v + gam * sp.apply_k(d, v)
    guesses = {
        "prev": H[n].copy(),
        "drift": gold[n] + (Un[n] - U[n]),
        "pdrift": gold[n] + pinv * (w @ (Un[: n + 1] - U[: n + 1])),
    }
    for k_, x0 in guesses.items():
        x, it = pcg(A, rhs, x0, pinv, 1e-13, 500, n)
        its[k_].append(it)
    Un[n + 1] = fold[n] + (x - gold[n])
for k_, v in its.items():
    print(f"{k_:7s} mean {np.mean(v):6.2f} per solve  {v}")
