"""Spatial operators for the oracle — TEST INFRASTRUCTURE ONLY.

``ChebyshevSpace`` restates ``pkg/src/parafrac/spectral.py`` (collocation
nodes, D1, Clenshaw-Curtis weights, ``assemble_diffusion``, ``l2_norm``) and
the inline batched assembly of ``stepping.py:219-237``.  ``Sine1D`` and
``Sine2D`` are the sine spectral-Galerkin operators of SURVEY.md §8.0, which
the reference does not contain; they plug into the same stepping algebra.

Every space exposes the same five hooks used by ``oracle.stepping``:

``initial_state(problem)``
    state at t=0 (nodal values or sine coefficients);
``operator(u, t, problem, batched)``
    the frozen-coefficient operator data at ``(u, t)``;
``source(u, t, problem, batched)``
    the load vector ``f`` seen by the right-hand side;
``solve(opdata, gam, rhs, step, batched)``
    the solution of ``(I + gam K) x = rhs`` (collocation: ``(I - gam A)``);
``norm(v)``
    the discrete L2 norm used by the driver's diff and guard.
"""

from __future__ import annotations

import math

import numpy as np
from scipy.linalg import lu_factor, lu_solve

from .errors import CoefficientError, SolverFailure

PIVOT_RTOL = 1e-14  # stepping.py:40


# --------------------------------------------------------------------------
# Chebyshev collocation (the reference operator)
# --------------------------------------------------------------------------

def clenshaw_curtis_weights(degree):
    """``spectral.py:27-45``."""
    n = degree
    j = np.arange(n + 1)
    ks = np.arange(1, n // 2 + 1)
    if ks.size:
        bcoef = np.where(2 * ks == n, 0.5, 1.0) * (2.0 / (4.0 * ks**2 - 1.0))
        w = (2.0 / n) * (1.0 - np.cos(2.0 * np.pi * np.outer(j, ks) / n) @ bcoef)
    else:
        w = np.full(n + 1, 2.0 / n)
    w[0] *= 0.5
    w[-1] *= 0.5
    return w


def _lu_solve_checked(system, rhs, step):
    """Dense LU with the pivot check (``stepping.py:62-75``)."""
    try:
        lu, piv = lu_factor(system, check_finite=False)
    except Exception as exc:  # pragma: no cover - LAPACK raises rarely
        raise SolverFailure(step, f"LU factorisation failed: {exc}") from exc
    scale = float(np.abs(system).max())
    pivot_min = float(np.abs(np.diag(lu)).min())
    if not np.isfinite(pivot_min) or pivot_min <= PIVOT_RTOL * scale:
        raise SolverFailure(step, "singular or ill-conditioned time-step system")
    out = lu_solve((lu, piv), rhs, check_finite=False)
    if not np.isfinite(out).all():
        raise SolverFailure(step, "non-finite solution from linear solve")
    return out


def _batched_solve(system, rhs, step):
    """Batched ``np.linalg.solve`` as in ``stepping.py:236-241``."""
    try:
        sol = np.linalg.solve(system, rhs[:, :, None])[:, :, 0]
    except np.linalg.LinAlgError as exc:
        raise SolverFailure(step, f"fine-sweep solve failed: {exc}") from exc
    if not np.isfinite(sol).all():
        raise SolverFailure(step, "non-finite solution in fine sweep")
    return sol


class ChebyshevSpace:
    """Chebyshev-Lobatto collocation on ``[a, b]`` (``spectral.py:48-103``)."""

    kind = "cheb1d"

    def __init__(self, degree, a=0.0, b=1.0):
        if degree < 2:
            raise ValueError("degree must be at least 2 so interior nodes exist")
        if not a < b:
            raise ValueError(f"invalid interval [{a}, {b}]")
        j = np.arange(degree + 1)
        xi = np.cos(np.pi * j / degree)
        csign = np.where((j == 0) | (j == degree), 2.0, 1.0) * (-1.0) ** j
        diff = xi[:, None] - xi[None, :]
        np.fill_diagonal(diff, 1.0)
        d1 = (csign[:, None] / csign[None, :]) / diff
        np.fill_diagonal(d1, 0.0)
        np.fill_diagonal(d1, -d1.sum(axis=1))
        d1 *= 2.0 / (b - a)
        self.degree = degree
        self.a = float(a)
        self.b = float(b)
        self.d1 = d1
        self.d2 = d1 @ d1
        self.nodes = 0.5 * (a + b) + 0.5 * (b - a) * xi
        self.quad_weights = clenshaw_curtis_weights(degree) * (0.5 * (b - a))
        self._eye = np.eye(degree - 1)

    @property
    def size(self):
        return self.degree - 1

    interior_size = size

    @property
    def interior_nodes(self):
        return self.nodes[1:-1]

    def initial_state(self, problem):
        """``stepping.py:51-54``."""
        u0 = np.asarray(problem.initial(self.interior_nodes), dtype=float)
        return np.broadcast_to(u0, (self.size,)).astype(float, copy=True)

    def operator(self, u, t, problem, batched):
        """Interior block of ``D1 diag(D) D1`` (``spectral.py:106-127``; batched
        form ``stepping.py:221-228``)."""
        npts = self.degree + 1
        if batched:
            bs = u.shape[0]
            full = np.zeros((bs, npts))
            full[:, 1:-1] = u
            dv = np.asarray(problem.diffusion(self.nodes[None, :], t[:, None], full), dtype=float)
            dv = np.broadcast_to(dv, (bs, npts))
            if not np.isfinite(dv).all():
                bad = int(np.flatnonzero(~np.isfinite(dv))[0] % npts)
                raise CoefficientError(bad, "diffusion coefficient is not finite")
            return ((self.d1 * dv[:, None, :]) @ self.d1)[:, 1:-1, 1:-1]
        full = np.zeros(npts)
        full[1:-1] = u
        dv = np.asarray(problem.diffusion(self.nodes, t, full), dtype=float)
        dv = np.broadcast_to(dv, self.nodes.shape)
        if not np.isfinite(dv).all():
            bad = int(np.flatnonzero(~np.isfinite(dv))[0])
            raise CoefficientError(bad, "diffusion coefficient is not finite")
        afull = (self.d1 * dv) @ self.d1
        return afull[1:-1, 1:-1]

    def source(self, u, t, problem, batched):
        """``stepping.py:57-59`` / ``:229-233``."""
        if batched:
            f = problem.source(self.interior_nodes[None, :], t[:, None], u)
            return np.broadcast_to(np.asarray(f, dtype=float), u.shape)
        f = np.asarray(problem.source(self.interior_nodes, t, u), dtype=float)
        return np.broadcast_to(f, (self.size,))

    def solve(self, a_int, gam, rhs, step, batched):
        """``system = I - gam*A`` (``stepping.py:111,235``)."""
        system = self._eye - gam * a_int
        if batched:
            return _batched_solve(system, rhs, step)
        return _lu_solve_checked(system, rhs, step)

    def norm(self, v):
        """Clenshaw-Curtis interior norm (``spectral.py:130-136``)."""
        v = np.asarray(v, dtype=float)
        return math.sqrt(float(np.dot(self.quad_weights[1:-1], np.square(v))))


def build_operator(degree, a=0.0, b=1.0):
    """``spectral.py:74`` — the reference's constructor name."""
    return ChebyshevSpace(degree, a, b)


# --------------------------------------------------------------------------
# PCG shared by the sine spaces (mirrors the device solver)
# --------------------------------------------------------------------------

def pcg(apply_a, rhs, x0, pinv, tol, maxit, step):
    """Preconditioned CG on one system, the exact recurrence the device runs.

    Stops when the recursively updated residual satisfies
    ``||r||_2 <= tol * ||rhs||_2``.  Returns ``(x, iterations)``.
    """
    x = x0.copy()
    rhs_norm = math.sqrt(float(np.dot(rhs.ravel(), rhs.ravel())))
    if rhs_norm == 0.0:
        return np.zeros_like(rhs), 0
    r = rhs - apply_a(x)
    thresh = tol * rhs_norm
    if math.sqrt(float(np.dot(r.ravel(), r.ravel()))) <= thresh:
        return x, 0
    z = pinv * r
    p = z.copy()
    rz = float(np.dot(r.ravel(), z.ravel()))
    for it in range(1, maxit + 1):
        q = apply_a(p)
        alpha = rz / float(np.dot(p.ravel(), q.ravel()))
        x = x + alpha * p
        r = r - alpha * q
        if math.sqrt(float(np.dot(r.ravel(), r.ravel()))) <= thresh:
            return x, it
        z = pinv * r
        rz_new = float(np.dot(r.ravel(), z.ravel()))
        beta = rz_new / rz
        rz = rz_new
        p = z + beta * p
    raise SolverFailure(step, "PCG did not converge")


# --------------------------------------------------------------------------
# Sine spectral Galerkin, 1-D
# --------------------------------------------------------------------------

class Sine1D:
    """Orthonormal basis ``sqrt(2) sin(k pi x)``, ``k=1..M`` on (0, 1).

    Quadrature: ``Q = 2M`` midpoints ``x_q = (q+1/2)/Q``, ``w_q = 1/Q``.
    ``K = S'^T diag(w D) S'`` and ``F = S^T (w f)`` at the previous substep;
    the system is ``(I + gam K) c = rhs`` (Galerkin K is SPD, hence ``+``).
    ``solver="direct"`` uses the batched LU / checked LU of the reference;
    ``solver="pcg"`` runs the device's PCG recurrence.
    """

    kind = "sine1d"

    def __init__(self, modes, solver="direct", pcg_tol=1e-14, pcg_maxit=500):
        if modes < 1:
            raise ValueError("need at least one mode")
        self.M = int(modes)
        self.Q = 2 * self.M
        q = np.arange(self.Q)
        self.x = (q + 0.5) / self.Q
        self.w = 1.0 / self.Q
        k = np.arange(1, self.M + 1)
        self.k = k.astype(float)
        self.S = math.sqrt(2.0) * np.sin(np.pi * np.outer(self.x, k))
        self.Sp = math.sqrt(2.0) * np.pi * k[None, :] * np.cos(np.pi * np.outer(self.x, k))
        self.solver = solver
        self.pcg_tol = pcg_tol
        self.pcg_maxit = pcg_maxit
        self.pcg_iterations = []
        self._eye = np.eye(self.M)

    @property
    def size(self):
        return self.M

    def initial_state(self, problem):
        coeffs = getattr(problem, "initial_coefficients", None)
        if coeffs is not None:
            c = np.asarray(coeffs(self.M), dtype=float)
            return c.copy()
        u0 = np.asarray(problem.initial(self.x), dtype=float)
        return (self.w * u0) @ self.S

    def grid_values(self, c):
        return c @ self.S.T

    def _dvals(self, u, t, problem, batched):
        x = self.x[None, :] if batched else self.x
        tt = t[:, None] if batched else t
        d = np.asarray(problem.diffusion(x, tt, u), dtype=float)
        d = np.broadcast_to(d, u.shape)
        if not np.isfinite(d).all():
            bad = int(np.flatnonzero(~np.isfinite(d))[0] % self.Q)
            raise CoefficientError(bad, "diffusion coefficient is not finite")
        return self.w * d

    def operator(self, c, t, problem, batched):
        u = self.grid_values(c)
        d = self._dvals(u, t, problem, batched)
        if self.solver == "pcg":
            return d
        if batched:
            return (self.Sp.T[None, :, :] * d[:, None, :]) @ self.Sp
        return (self.Sp.T * d[None, :]) @ self.Sp

    def source(self, c, t, problem, batched):
        u = self.grid_values(c)
        x = self.x[None, :] if batched else self.x
        tt = t[:, None] if batched else t
        g = np.asarray(problem.source(x, tt, u), dtype=float)
        g = np.broadcast_to(g, u.shape)
        return (self.w * g) @ self.S

    def apply_k(self, d, v):
        return ((v @ self.Sp.T) * d) @ self.Sp

    def solve(self, opdata, gam, rhs, step, batched, x0=None):
        if self.solver == "pcg":
            return self._solve_pcg(opdata, gam, rhs, step, batched, x0)
        system = self._eye + gam * opdata
        if batched:
            return _batched_solve(system, rhs, step)
        return _lu_solve_checked(system, rhs, step)

    def _solve_pcg(self, d, gam, rhs, step, batched, x0):
        if not batched:
            d, rhs = d[None], rhs[None]
            x0 = None if x0 is None else x0[None]
        out = np.empty_like(rhs)
        for i in range(rhs.shape[0]):
            di = d[i]
            dbar = float(np.sum(di))
            pinv = 1.0 / (1.0 + gam * dbar * np.pi**2 * self.k**2)
            start = rhs[i] * 0.0 if x0 is None else x0[i]
            out[i], its = pcg(lambda v: v + gam * self.apply_k(di, v), rhs[i], start, pinv,
                              self.pcg_tol, self.pcg_maxit, step)
            self.pcg_iterations.append(its)
        return out if batched else out[0]

    def norm(self, v):
        v = np.asarray(v, dtype=float)
        return math.sqrt(float(np.dot(v, v)))


# --------------------------------------------------------------------------
# Sine spectral Galerkin, 2-D tensor basis
# --------------------------------------------------------------------------

class Sine2D:
    """Tensor basis ``2 sin(k1 pi x) sin(k2 pi y)``; states are ``C.ravel()``.

    Grid values ``U = S C S^T`` on the ``Q x Q`` midpoint grid; the operator
    is applied matrix-free,
    ``K C = S'^T (W d (S' C S^T)) S + S^T (W d (S C S'^T)) S'``, and every
    solve is PCG with ``P^-1 = 1/(1 + gam dbar pi^2 (k1^2 + k2^2))``,
    ``dbar = sum(W d)``, initial guess the previous state.
    """

    kind = "sine2d"

    def __init__(self, modes, pcg_tol=1e-13, pcg_maxit=500):
        self.M = int(modes)
        self.Q = 2 * self.M
        one = Sine1D(self.M)
        self.x = one.x
        self.S = one.S
        self.Sp = one.Sp
        self.w = one.w * one.w
        k = one.k
        self.k2 = (k[:, None] ** 2 + k[None, :] ** 2)
        self.pcg_tol = pcg_tol
        self.pcg_maxit = pcg_maxit
        self.pcg_iterations = []
        self.X1, self.X2 = np.meshgrid(self.x, self.x, indexing="ij")

    @property
    def size(self):
        return self.M * self.M

    def initial_state(self, problem):
        coeffs = getattr(problem, "initial_coefficients", None)
        if coeffs is not None:
            return np.asarray(coeffs(self.M), dtype=float).reshape(-1).copy()
        u0 = np.asarray(problem.initial((self.X1, self.X2)), dtype=float)
        return (self.S.T @ (self.w * u0) @ self.S).reshape(-1)

    def grid_values(self, c):
        C = c.reshape(c.shape[:-1] + (self.M, self.M))
        return self.S @ C @ self.S.T

    def operator(self, c, t, problem, batched):
        U = self.grid_values(c)
        if batched:
            x = (self.X1[None], self.X2[None])
            tt = t[:, None, None]
        else:
            x = (self.X1, self.X2)
            tt = t
        d = np.asarray(problem.diffusion(x, tt, U), dtype=float)
        d = np.broadcast_to(d, U.shape)
        if not np.isfinite(d).all():
            bad = int(np.flatnonzero(~np.isfinite(d))[0] % (self.Q * self.Q))
            raise CoefficientError(bad, "diffusion coefficient is not finite")
        return self.w * d

    def source(self, c, t, problem, batched):
        U = self.grid_values(c)
        if batched:
            x = (self.X1[None], self.X2[None])
            tt = t[:, None, None]
        else:
            x = (self.X1, self.X2)
            tt = t
        g = np.broadcast_to(np.asarray(problem.source(x, tt, U), dtype=float), U.shape)
        F = self.S.T @ (self.w * g) @ self.S
        return F.reshape(F.shape[:-2] + (self.M * self.M,))

    def apply_k(self, d, v):
        C = v.reshape(self.M, self.M)
        gx = self.Sp @ C @ self.S.T
        gy = self.S @ C @ self.Sp.T
        out = self.Sp.T @ (d * gx) @ self.S + self.S.T @ (d * gy) @ self.Sp
        return out.reshape(-1)

    def solve(self, d, gam, rhs, step, batched, x0=None):
        if not batched:
            d, rhs = d[None], rhs[None]
            x0 = None if x0 is None else x0[None]
        out = np.empty_like(rhs)
        for i in range(rhs.shape[0]):
            di = d[i]
            dbar = float(np.sum(di))
            pinv = (1.0 / (1.0 + gam * dbar * np.pi**2 * self.k2)).reshape(-1)
            start = rhs[i] * 0.0 if x0 is None else x0[i]
            out[i], its = pcg(lambda v: v + gam * self.apply_k(di, v), rhs[i], start, pinv,
                              self.pcg_tol, self.pcg_maxit, step)
            self.pcg_iterations.append(its)
        return out if batched else out[0]

    def norm(self, v):
        v = np.asarray(v, dtype=float).ravel()
        return math.sqrt(float(np.dot(v, v)))
