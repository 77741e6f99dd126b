"""CPU study: PCG iterations in the first substeps of a slice (config 3, 1-D)
for initial guesses that use the slice's end state U[n+1] (the coarse
prediction the sweep already has) besides the slice's own recent states.

    python slice_start_guess.py [n] [m]
"""
import sys, time
import numpy as np
sys.path.insert(0, "/root/repo")
import oracle
from oracle import problems as OP
from oracle.spaces import pcg
from oracle.weights import weights_for, gamma_2_minus
from oracle.stepping import coarse_contribution

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
m = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
M, P, alpha, T = 512, 64, 0.3, 2.0
prob = OP.config(3); sp = oracle.Sine1D(M)
grids = oracle.TimeGrids(T, P, m)
dt = grids.dt
gam = dt**alpha * gamma_2_minus(alpha)
rows = weights_for(alpha).fine_rows(m)
U = oracle.run_coarse(prob, sp, grids)
contrib = coarse_contribution(weights_for(alpha), U[: n + 1], n, m, alpha)
path = np.empty((m + 1, M)); path[0] = U[n]
C = [[1], [2, -1], [3, -3, 1], [4, -6, 4, -1], [5, -10, 10, -5, 1], [6, -15, 20, -15, 6, -1]]
tau = lambda k: ((n * m + k) * dt) ** alpha
def interp(k):  # coarse-chord in tau between U[n] (k=0) and U[n+1] (k=m)
    w = (tau(k) - tau(0)) / (tau(m) - tau(0))
    return U[n] + w * (U[n + 1] - U[n])
def poly(r, order, f=lambda k: path[k]):
    p = min(order, r - 1)
    return sum(C[p][j] * f(r - 1 - j) for j in range(p + 1))
def lag_weights(nodes, target):
    w = []
    for j in range(len(nodes)):
        v = 1.0
        for q in range(len(nodes)):
            if q != j:
                v *= (target - nodes[q]) / (nodes[j] - nodes[q])
        w.append(v)
    return np.array(w)
def tau_local(r, order):  # Lagrange in the slice's own tau = (r dt)^alpha
    p = min(order, r - 1)
    ks = np.arange(r - 1, r - 2 - p, -1)
    w = lag_weights([(k * dt) ** alpha for k in ks], (r * dt) ** alpha)
    return w @ path[ks]
cands = {
    "poly5": lambda r: poly(r, 5),
    "tloc3": lambda r: tau_local(r, 3),
    "tloc5": lambda r: tau_local(r, 5),
    "tloc7": lambda r: tau_local(r, 7),
    "chord": lambda r: interp(r),
    "chord+dev5": lambda r: interp(r) + poly(r, 5, lambda k: path[k] - interp(k)),
    "chord+dev2": lambda r: interp(r) + poly(r, 2, lambda k: path[k] - interp(k)),
    "chord+dev0": lambda r: interp(r) + (path[r - 1] - interp(r - 1)),
}
its = {k: [] for k in cands}
last = min(m, 128)
for r in range(1, last + 1):
    t_prev = n * m * dt + (r - 1) * dt
    u_prev = path[r - 1]
    K = sp.operator(u_prev, t_prev, prob, batched=False)
    F = sp.source(u_prev, t_prev, prob, batched=False)
    rhs = rows[r - 1][:r] @ path[:r] + gam * F + contrib[r - 1]
    A = np.eye(M) + gam * K
    path[r] = np.linalg.solve(A, rhs)
    d = sp._dvals(sp.grid_values(u_prev), t_prev, prob, False)
    pinv = 1.0 / (1.0 + gam * float(np.sum(d)) * np.pi**2 * sp.k**2)
    for name, fn in cands.items():
        _, it = pcg(lambda v: A @ v, rhs, fn(r), pinv, 1e-14, 60, (n, r))
        its[name].append(it)
edges = [1, 2, 4, 8, 16, 32, 64, last + 1]
print(f"slice {n}, m={m}: PCG iterations per substep range")
print("range       " + " ".join(f"{k:>11s}" for k in its))
for a, b in zip(edges[:-1], edges[1:]):
    print(f"[{a:3d},{b:3d})  " + " ".join(f"{np.mean(v[a-1:b-1]):11.2f}" for v in its.values()))
print("total      " + " ".join(f"{np.sum(v):11d}" for v in its.values()))
