"""Reference-compatible solver API on the B200 path.

Same names, arguments, return values and exceptions as ``parafrac``
(``stepping.py:87-288``, ``parareal.py:32-189``); every function below calls
the C-ABI (``include/parafrac_b200.h``) and runs sm_100a kernels.  ``threads``
is accepted for signature compatibility and ignored: the device batches every
slice of a sweep at once, and results do not depend on any split
(``test_stepping.py:166-175``).
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from ._lib import context_for, f64, lib, ptr
from .spaces import initial_state, l2_norm

__all__ = ["PararealIterate", "PararealReport", "chain_fine", "coarse_step", "exactness_check",
           "fine_propagate", "fine_sweep_intervals", "parareal_solve", "run_coarse",
           "run_fine_sequential"]

START_MISMATCH_TOL = 1e-10  # stepping.py:41


@dataclass
class PararealIterate:
    """``parareal.py:32-45``: ``states[n+1] == fine_endpoints[n] + (coarse_new[n] - coarse_old[n])``."""

    k: int
    states: np.ndarray
    coarse_new: np.ndarray
    coarse_old: np.ndarray
    fine_endpoints: np.ndarray


@dataclass
class PararealReport:
    """``parareal.py:48-59`` plus device statistics."""

    iterations: int
    diffs: list
    stop_reason: str
    threads: int
    wall_time: float
    iteration_times: list = field(default_factory=list)
    errors_vs_reference: Optional[list] = None
    wall_time_reference: Optional[float] = None
    device_stats: Optional[dict] = None


def coarse_step(history, op, grids, problem, step_index=None):
    """One coarse L1 step with the full coarse history (``stepping.py:87-112``)."""
    states = np.asarray(history, dtype=float)
    if states.ndim == 1:
        states = states[None, :]
    if states.ndim != 2 or states.shape[0] < 1 or states.shape[1] != op.interior_size:
        raise ValueError("history must be a nonempty stack of interior-node states")
    n = states.shape[0] - 1
    if step_index is None:
        step_index = n
    ctx = context_for(problem, op, grids)
    states = f64(states)
    out = np.empty(op.interior_size)
    with ctx.lock:
        ctx.check(lib.pf_coarse_step(ctx.handle, ptr(states), n + 1, int(step_index), ptr(out)),
                  default_step=step_index)
    return out


def run_coarse(problem, op, grids):
    """Sequential coarse trajectory (``stepping.py:115-121``), one device kernel."""
    ctx = context_for(problem, op, grids)
    u0 = f64(initial_state(problem, op))
    traj = np.empty((grids.nt + 1, op.interior_size))
    with ctx.lock:
        ctx.check(lib.pf_run_coarse(ctx.handle, ptr(u0), ptr(traj)))
    return traj


def fine_propagate(start, coarse_history, op, grids, problem):
    """One slice of the hybrid fine march (``stepping.py:142-186``); returns
    ``(endpoint, fine_path)`` with ``fine_path[r-1]`` the state at ``(n, r)``."""
    hist = np.asarray(coarse_history, dtype=float)
    if hist.ndim == 1:
        hist = hist[None, :]
    start = np.asarray(start, dtype=float)
    if hist.shape[1] != op.interior_size or start.shape != (op.interior_size,):
        raise ValueError("states must be vectors of interior-node values")
    n = hist.shape[0] - 1
    scale = max(1.0, float(np.abs(start).max()))
    if float(np.abs(hist[n] - start).max()) > START_MISMATCH_TOL * scale:
        raise ValueError("start state disagrees with the last coarse history entry")
    ctx = context_for(problem, op, grids)
    hist = f64(hist)
    start = f64(start)
    endpoint = np.empty(op.interior_size)
    path = np.empty((grids.m, op.interior_size))
    with ctx.lock:
        # path[0] = start (stepping.py:170-171): within START_MISMATCH_TOL of hist[n], not equal
        ctx.check(lib.pf_fine_propagate(ctx.handle, ptr(start), ptr(hist), n + 1, ptr(endpoint), ptr(path)))
    return endpoint, path


def fine_sweep_intervals(u_nodes, n_lo, n_hi, op, grids, problem):
    """Fine endpoints of slices ``n_lo..n_hi-1`` marched together (``stepping.py:189-243``).

    THE hot path: one kernel launch, one CTA per slice, all ``m`` substeps
    inside the kernel.
    """
    U = np.asarray(u_nodes)
    bs = n_hi - n_lo
    if bs < 1 or n_hi > U.shape[0] - 1:
        raise ValueError("interval range outside the supplied coarse states")
    ctx = context_for(problem, op, grids)
    U = f64(U)
    out = np.empty((bs, op.interior_size))
    with ctx.lock:
        ctx.check(lib.pf_fine_sweep(ctx.handle, ptr(U), U.shape[0], int(n_lo), int(n_hi), ptr(out)))
    return out


def chain_fine(problem, op, grids):
    """The parareal fixed point, fine propagator chained slice by slice (``stepping.py:246-257``)."""
    ctx = context_for(problem, op, grids)
    u0 = f64(initial_state(problem, op))
    traj = np.empty((grids.nt + 1, op.interior_size))
    with ctx.lock:
        ctx.check(lib.pf_chain_fine(ctx.handle, ptr(u0), ptr(traj)))
    return traj


def run_fine_sequential(problem, op, grids):
    """Full-history serial solver (``stepping.py:260-288``); returns ``(states, seconds)``."""
    t0 = time.perf_counter()
    ctx = context_for(problem, op, grids)
    u0 = f64(initial_state(problem, op))
    states = np.empty((grids.nt + 1, op.interior_size))
    with ctx.lock:
        ctx.check(lib.pf_fine_sequential(ctx.handle, ptr(u0), ptr(states)))
    return states, time.perf_counter() - t0


def _solve(problem, op, grids, tol, k_max, threads, reference):
    """``parareal.py:91-155`` on device: run_coarse, then per iteration one
    fine-sweep launch and one correction-sweep launch (guards + diff fused)."""
    t0 = time.perf_counter()
    ctx = context_for(problem, op, grids)
    nt, ni = grids.nt, op.interior_size
    u0 = f64(initial_state(problem, op))
    states = np.empty((nt + 1, ni))
    g_new = np.empty((nt, ni))
    g_old = np.empty((nt, ni))
    f_old = np.empty((nt, ni))
    diffs = np.zeros(k_max)
    times = np.zeros(k_max)
    errors = np.zeros(k_max + 1) if reference is not None else None
    ref = f64(reference) if reference is not None else None
    iters = _lib.C.c_int(0)
    stop = _lib.C.c_int(0)
    with ctx.lock:
        lib.pf_reset_stats(ctx.handle)
        ctx.check(lib.pf_parareal(ctx.handle, ptr(u0), float(tol) if tol is not None else -1.0, int(k_max),
                                  ptr(ref), ptr(states), ptr(g_new), ptr(g_old), ptr(f_old), ptr(diffs),
                                  ptr(times), ptr(errors), _lib.C.byref(iters), _lib.C.byref(stop)))
        stats = ctx.stats()
    k = iters.value
    iterate = PararealIterate(k=k, states=states, coarse_new=g_new, coarse_old=g_old, fine_endpoints=f_old)
    report = PararealReport(
        iterations=k,
        diffs=[float(d) for d in diffs[:k]],
        stop_reason="tol" if stop.value == 1 else "k_max",
        threads=threads,
        wall_time=time.perf_counter() - t0,
        iteration_times=[float(t) for t in times[:k]],
        errors_vs_reference=None if errors is None else [float(e) for e in errors[: k + 1]],
        device_stats=stats,
    )
    return iterate, report


def parareal_solve(problem, op, grids, tol=1e-10, k_max=20, threads=1, reference=None):
    """``parareal.py:158-172``: returns ``(PararealIterate, PararealReport)``."""
    if not tol > 0:
        raise ValueError("tolerance must be positive")
    if k_max < 1:
        raise ValueError("k_max must be at least 1")
    if threads < 1:
        raise ValueError("threads must be at least 1")
    return _solve(problem, op, grids, tol, int(k_max), int(threads), reference)


def exactness_check(problem, op, grids, k):
    """Finite termination: max L2 gap of iterate ``k`` to ``chain_fine`` on nodes ``0..k``
    (``parareal.py:175-189``)."""
    if not 0 <= k <= grids.nt:
        raise ValueError(f"iteration count k={k} outside 0..{grids.nt}")
    if k == 0:
        return 0.0
    fixed = chain_fine(problem, op, grids)
    iterate, _ = _solve(problem, op, grids, tol=None, k_max=k, threads=1, reference=None)
    return max(l2_norm(op, iterate.states[n] - fixed[n]) for n in range(k + 1))
