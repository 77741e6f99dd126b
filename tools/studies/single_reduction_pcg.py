"""Numpy trace: single-reduction PCG (rr, rz from the recurrences) vs the true residual on config-1 systems (cold start: the recurrence error stays at eps x the initial rr, so the 1e-14 tolerance is unreachable and the solve diverges)."""
import math, sys, numpy as np
sys.path.insert(0, "/root/repo")
import oracle
from oracle import problems as OP
from oracle.weights import weights_for, gamma_2_minus

def pcg_single(A, rhs, x0, pinv, tol, maxit):
    x = x0.copy(); bb = rhs @ rhs
    r = rhs - A @ x; z = pinv * r; p = z.copy()
    rr = r @ r; rz = r @ z; thr = tol * tol * bb
    if not rr > thr: return x, 0, "ok"
    for it in range(1, maxit + 1):
        q = A @ p
        pq, rq, qq, zq, qPq = p @ q, r @ q, q @ q, z @ q, q @ (pinv * q)
        a = rz / pq
        x = x + a * p; r = r - a * q; z = pinv * r
        rr = rr - 2 * a * rq + a * a * qq
        rzn = rz - 2 * a * zq + a * a * qPq
        if not rr > thr: return x, it, "ok"
        b = rzn / rz; rz = rzn; p = z + b * p
    return x, maxit, f"maxit rr={rr:.3e} thr={thr:.3e} true={r@r:.3e} rz={rz:.3e}"

M, P, m = 32, 8, 64
prob = OP.config(1); sp = oracle.Sine1D(M)
dt = 1.0 / (P * m); alpha = 0.5
gam = dt**alpha * gamma_2_minus(alpha)
rows = weights_for(alpha).fine_rows(m)
path = np.empty((m + 1, M)); path[0] = sp.initial_state(prob)
for r in range(1, m + 1):
    t_prev = (r - 1) * dt; u_prev = path[r - 1]
    K = sp.operator(u_prev, t_prev, prob, batched=False)
    F = sp.source(u_prev, t_prev, prob, batched=False)
    rhs = rows[r - 1][:r] @ path[:r] + gam * F
    A = np.eye(M) + gam * K
    path[r] = np.linalg.solve(A, rhs)
    d = sp._dvals(sp.grid_values(u_prev), t_prev, prob, False)
    pinv = 1.0 / (1.0 + gam * float(np.sum(d)) * np.pi**2 * sp.k**2)
    x0 = u_prev
    x, it, msg = pcg_single(A, rhs, x0, pinv, 1e-14, 60)
    if msg != "ok" or r < 4: print(r, it, msg, np.linalg.norm(x - path[r]) / np.linalg.norm(path[r]))
# debug one system
r = 2
t_prev = (r - 1) * dt; u_prev = path[r - 1]
K = sp.operator(u_prev, t_prev, prob, batched=False)
F = sp.source(u_prev, t_prev, prob, batched=False)
rhs = rows[r - 1][:r] @ path[:r] + gam * F
A = np.eye(M) + gam * K
d = sp._dvals(sp.grid_values(u_prev), t_prev, prob, False)
pinv = 1.0 / (1.0 + gam * float(np.sum(d)) * np.pi**2 * sp.k**2)
x = u_prev.copy(); rv = rhs - A @ x; z = pinv * rv; p = z.copy(); rr = rv @ rv; rz = rv @ z
for it in range(6):
    q = A @ p; pq = p @ q; a = rz / pq
    rq, qq, zq, qPq = rv @ q, q @ q, z @ q, q @ (pinv * q)
    rvn = rv - a * q
    print(it, "rr formula", rr - 2*a*rq + a*a*qq, "true", rvn @ rvn, "rz formula", rz - 2*a*zq + a*a*qPq, "true", rvn @ (pinv*rvn), "pq", pq)
    rv = rvn; z = pinv * rv; rzn = rv @ z; p = z + (rzn / rz) * p; rz = rzn; rr = rv @ rv
print("---- pcg_single trace")
def trace(A, rhs, x0, pinv, tol, maxit):
    x = x0.copy(); bb = rhs @ rhs
    r = rhs - A @ x; z = pinv * r; p = z.copy()
    rr = r @ r; rz = r @ z; thr = tol * tol * bb
    for it in range(1, maxit + 1):
        q = A @ p
        pq, rq, qq, zq, qPq = p @ q, r @ q, q @ q, z @ q, q @ (pinv * q)
        a = rz / pq
        x = x + a * p; r = r - a * q; z = pinv * r
        rr = rr - 2 * a * rq + a * a * qq
        rzn = rz - 2 * a * zq + a * a * qPq
        print(it, rr, r @ r, rzn, r @ z)
        b = rzn / rz; rz = rzn; p = z + b * p
trace(A, rhs, u_prev, pinv, 1e-14, 5)
