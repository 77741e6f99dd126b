"""CPU study (oracle's exact path): relative residual of polynomial extrapolation guesses of order
5..10 in the steady part of a slice (config 3), against the PCG tolerance 1e-14 -- can a higher
order make the guess itself pass (zero iterations)?   python steady_guess_order.py [n] [rmax]"""
import sys
from math import comb
import numpy as np
sys.path.insert(0, "/root/repo")
import oracle
from oracle import problems as OP
from oracle.weights import weights_for, gamma_2_minus
from oracle.stepping import coarse_contribution

n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
rmax = int(sys.argv[2]) if len(sys.argv) > 2 else 260
m = 1024
M, P, alpha, T = 512, 64, 0.3, 2.0
prob = OP.config(3); sp = oracle.Sine1D(M)
grids = oracle.TimeGrids(T, P, m)
dt = grids.dt
gam = dt**alpha * gamma_2_minus(alpha)
rows = weights_for(alpha).fine_rows(m)
U = oracle.run_coarse(prob, sp, grids)
contrib = coarse_contribution(weights_for(alpha), U[: n + 1], n, m, alpha)
path = np.empty((rmax + 1, M)); path[0] = U[n]
orders = [5, 6, 7, 8, 9, 10, 12]
res = {p: [] for p in orders}
for r in range(1, rmax + 1):
    t_prev = n * m * dt + (r - 1) * dt
    u_prev = path[r - 1]
    K = sp.operator(u_prev, t_prev, prob, batched=False)
    F = sp.source(u_prev, t_prev, prob, batched=False)
    rhs = rows[r - 1][:r] @ path[:r] + gam * F + contrib[r - 1]
    A = np.eye(M) + gam * K
    path[r] = np.linalg.solve(A, rhs)
    for p in orders:
        q = min(p, r - 1)
        g = sum((-1) ** j * comb(q + 1, j + 1) * path[r - 1 - j] for j in range(q + 1))
        res[p].append(np.linalg.norm(rhs - A @ g) / np.linalg.norm(rhs))
print(f"slice {n}: relative residual of the order-p polynomial guess (PCG tolerance 1e-14)")
print("  r range    " + " ".join(f"p={p:<8d}" for p in orders))
for a, b in [(17, 33), (33, 65), (65, 129), (129, 193), (193, rmax + 1)]:
    if a <= rmax:
        print(f"[{a:4d},{b:4d}) " + " ".join(f"{np.exp(np.mean(np.log(res[p][a - 1:b - 1]))):.2e}  " for p in orders))
