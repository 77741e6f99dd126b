"""CPU study: PCG iterations of slice 0 (config 3) for different initial-guess rules.

Marches slice 0 with the oracle's dense solve (the exact path), and at every
substep counts the iterations the device PCG recurrence (oracle.spaces.pcg,
tol 1e-14) needs from each candidate guess.  Usage: python slice0_guess.py [m]
"""
import math, sys, time
import numpy as np
sys.path.insert(0, "/root/repo")
import oracle
from oracle import problems as OP
from oracle.spaces import pcg
from oracle.weights import weights_for, gamma_2_minus

m = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
n = int(sys.argv[2]) if len(sys.argv) > 2 else 0
M, P, alpha, T = 512, 64, 0.3, 2.0
prob = OP.config(3)
sp = oracle.Sine1D(M)
dt = T / (P * m)
gam = dt**alpha * gamma_2_minus(alpha)
rows = weights_for(alpha).fine_rows(m)
path = np.empty((m + 1, M))
grids = oracle.TimeGrids(T, P, m)
U = oracle.run_coarse(prob, sp, grids)
from oracle.stepping import coarse_contribution
contrib = coarse_contribution(weights_for(alpha), U[: n + 1], n, m, alpha)
path[0] = U[n]

def lag_weights(nodes, target):
    w = []
    for j in range(len(nodes)):
        v = 1.0
        for q in range(len(nodes)):
            if q != j:
                v *= (target - nodes[q]) / (nodes[j] - nodes[q])
        w.append(v)
    return np.array(w)

def guess(r, order, var="tau", npts=None):
    p = min(order, r - 1)
    npt = p + 1 if npts is None else min(npts, r)
    ks = np.arange(r - 1, r - 1 - npt, -1)
    f = (lambda k: ((n * m + k) * dt) ** alpha) if var == "tau" else (lambda k: float(k))
    x = np.array([f(k) for k in ks]); tgt = f(r)
    if npt == p + 1:
        w = lag_weights(x, tgt)
    else:  # least squares polynomial of degree p through n points, evaluated at tgt
        V = np.vander(x - tgt, p + 1, increasing=True)
        w = np.linalg.pinv(V)[0]
    return w @ path[ks]

cands = {f"tau{o}": dict(order=o) for o in range(2, 9)}
cands.update({f"t{o}": dict(order=o, var="t") for o in (3, 4, 5)})
its = {k: [] for k in cands}
t0 = time.time()
for r in range(1, m + 1):
    t_prev = n * m * dt + (r - 1) * dt
    u_prev = path[r - 1]
    K = sp.operator(u_prev, t_prev, prob, batched=False)
    F = sp.source(u_prev, t_prev, prob, batched=False)
    rhs = rows[r - 1][:r] @ path[:r] + gam * F + contrib[r - 1]
    A = np.eye(M) + gam * K
    path[r] = np.linalg.solve(A, rhs)
    d = sp._dvals(sp.grid_values(u_prev), t_prev, prob, False)
    dbar = float(np.sum(d))
    pinv = 1.0 / (1.0 + gam * dbar * np.pi**2 * sp.k**2)
    for name, kw in cands.items():
        x0 = guess(r, **kw) if r >= 2 else u_prev
        _, it = pcg(lambda v: A @ v, rhs, x0, pinv, 1e-14, 50, (0, r))
        its[name].append(it)
print(f"slice {n}, m={m}, {time.time()-t0:.0f} s")
edges = [1, 4, 8, 16, 32, 64, 128, 256, 512, m + 1]
print("range      " + " ".join(f"{n:>7s}" for n in its))
for a, b in zip(edges[:-1], edges[1:]):
    print(f"[{a:4d},{b:4d}) " + " ".join(f"{np.mean(v[a-1:b-1]):7.3f}" for v in its.values()))
print("mean       " + " ".join(f"{np.mean(v):7.3f}" for v in its.values()))
best = sum(min(np.sum(v[a-1:b-1]) for v in its.values()) for a, b in zip(edges[:-1], edges[1:]))
print("best-per-range mean", best / m)
