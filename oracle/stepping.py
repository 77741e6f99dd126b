"""Propagators — restatement of ``pkg/src/parafrac/stepping.py`` (oracle, test infra).

The time-stepping algebra is the reference's line for line; only the
spatial hooks (``space.operator/source/solve``) are pluggable.  With
``ChebyshevSpace`` every array operation here is the one the reference
performs, so results agree bit for bit on this host.
"""

from __future__ import annotations

import time

import numpy as np

from .weights import gamma_2_minus, history_weights, weights_for

START_MISMATCH_TOL = 1e-10  # stepping.py:41


def _solve(space, opdata, gam, rhs, step, batched, x0):
    if getattr(space, "kind", "") == "cheb1d" or getattr(space, "solver", "pcg") == "direct":
        return space.solve(opdata, gam, rhs, step, batched)
    return space.solve(opdata, gam, rhs, step, batched, x0=x0)


def coarse_step(history, space, grids, problem, step_index=None):
    """One coarse L1 step with the full coarse history (``stepping.py:87-112``)."""
    states = np.asarray(history, dtype=float)
    if states.ndim == 1:
        states = states[None, :]
    if states.ndim != 2 or states.shape[0] < 1 or states.shape[1] != space.size:
        raise ValueError("history must be a nonempty stack of states")
    n = states.shape[0] - 1
    if step_index is None:
        step_index = n
    alpha = problem.alpha
    b = weights_for(alpha).on_grid(1, n + 2)
    w = history_weights(b, n)
    t_n = n * grids.dT
    u_n = states[n]
    gam = grids.dT**alpha * gamma_2_minus(alpha)
    opdata = space.operator(u_n, t_n, problem, batched=False)
    rhs = w @ states + gam * space.source(u_n, t_n, problem, batched=False)
    return _solve(space, opdata, gam, rhs, step_index, False, u_n)


def run_coarse(problem, space, grids):
    """Sequential coarse trajectory (``stepping.py:115-121``)."""
    traj = np.empty((grids.nt + 1, space.size))
    traj[0] = space.initial_state(problem)
    for n in range(grids.nt):
        traj[n + 1] = coarse_step(traj[: n + 1], space, grids, problem, step_index=n)
    return traj


def coarse_contribution(wt, hist, n, m, alpha):
    """Coarse-history bracket, one row per substep (``stepping.py:124-139``)."""
    ni = hist.shape[1]
    if n == 0:
        return np.zeros((m, ni))
    bq = wt.on_grid(m, n * m + 1)
    picks = bq[1 : n * m + 1].reshape(n, m)
    increments = hist[1:] - hist[:-1]
    return -(float(m) ** (-alpha)) * (picks.T @ increments[::-1])


def fine_propagate(start, coarse_history, space, grids, problem):
    """One slice of the hybrid fine march (``stepping.py:142-186``)."""
    hist = np.asarray(coarse_history, dtype=float)
    if hist.ndim == 1:
        hist = hist[None, :]
    start = np.asarray(start, dtype=float)
    if hist.shape[1] != space.size or start.shape != (space.size,):
        raise ValueError("states must be vectors of the space's size")
    n = hist.shape[0] - 1
    scale = max(1.0, float(np.abs(start).max()))
    if float(np.abs(hist[n] - start).max()) > START_MISMATCH_TOL * scale:
        raise ValueError("start state disagrees with the last coarse history entry")
    m = grids.m
    alpha = problem.alpha
    wt = weights_for(alpha)
    rows = wt.fine_rows(m)
    contrib = coarse_contribution(wt, hist, n, m, alpha)
    gam = grids.dt**alpha * gamma_2_minus(alpha)
    base_t = n * grids.dT
    path = np.empty((m + 1, space.size))
    path[0] = start
    for r in range(1, m + 1):
        t_prev = base_t + (r - 1) * grids.dt
        u_prev = path[r - 1]
        opdata = space.operator(u_prev, t_prev, problem, batched=False)
        rhs = (
            np.einsum("j,js->s", rows[r - 1], path[:r])
            + gam * space.source(u_prev, t_prev, problem, batched=False)
            + contrib[r - 1]
        )
        path[r] = _solve(space, opdata, gam, rhs, (n, r), False, u_prev)
    return path[m].copy(), path[1:].copy()


def fine_sweep_intervals(u_nodes, n_lo, n_hi, space, grids, problem, substeps=None):
    """Batched fine endpoints for slices ``n_lo..n_hi-1`` (``stepping.py:189-243``).

    ``substeps`` (oracle extension, default ``m``) stops the march early and
    returns the states after that many substeps; the CPU baseline uses it to
    time a bounded sample of the sweep.
    """
    U = np.asarray(u_nodes)
    bs = n_hi - n_lo
    if bs < 1 or n_hi > U.shape[0] - 1:
        raise ValueError("interval range outside the supplied coarse states")
    m = grids.m
    last = m if substeps is None else int(substeps)
    ni = space.size
    alpha = problem.alpha
    wt = weights_for(alpha)
    rows = wt.fine_rows(m)
    gam = grids.dt**alpha * gamma_2_minus(alpha)

    contrib = np.empty((bs, m, ni))
    for idx, n in enumerate(range(n_lo, n_hi)):
        contrib[idx] = coarse_contribution(wt, U[: n + 1], n, m, alpha)

    paths = np.empty((bs, m + 1, ni))
    paths[:, 0] = U[n_lo:n_hi]
    tn = np.arange(n_lo, n_hi) * grids.dT
    for r in range(1, last + 1):
        t_prev = tn + (r - 1) * grids.dt
        u_prev = paths[:, r - 1]
        opdata = space.operator(u_prev, t_prev, problem, batched=True)
        f_vec = space.source(u_prev, t_prev, problem, batched=True)
        rhs = np.einsum("j,bjs->bs", rows[r - 1], paths[:, :r]) + gam * f_vec + contrib[:, r - 1]
        paths[:, r] = _solve(space, opdata, gam, rhs, (n_lo, r), True, u_prev)
    return paths[:, last].copy()


def chain_fine(problem, space, grids):
    """The parareal fixed point (``stepping.py:246-257``)."""
    traj = np.empty((grids.nt + 1, space.size))
    traj[0] = space.initial_state(problem)
    for n in range(grids.nt):
        traj[n + 1] = fine_propagate(traj[n], traj[: n + 1], space, grids, problem)[0]
    return traj


def run_fine_sequential(problem, space, grids):
    """Full-history serial fine solver (``stepping.py:260-288``)."""
    t0 = time.perf_counter()
    total = grids.total_fine
    ni = space.size
    alpha = problem.alpha
    b = weights_for(alpha).on_grid(1, total + 1)
    dflip = np.ascontiguousarray((b[:-1] - b[1:])[::-1])
    gam = grids.dt**alpha * gamma_2_minus(alpha)
    hist = np.empty((total + 1, ni))
    hist[0] = space.initial_state(problem)
    for jj in range(1, total + 1):
        t_prev = (jj - 1) * grids.dt
        u_prev = hist[jj - 1]
        opdata = space.operator(u_prev, t_prev, problem, batched=False)
        rhs_hist = b[jj - 1] * hist[0]
        if jj >= 2:
            rhs_hist = rhs_hist + dflip[total - jj + 1 :] @ hist[1:jj]
        rhs = rhs_hist + gam * space.source(u_prev, t_prev, problem, batched=False)
        hist[jj] = _solve(space, opdata, gam, rhs, jj - 1, False, u_prev)
    states = hist[:: grids.m].copy()
    return states, time.perf_counter() - t0
