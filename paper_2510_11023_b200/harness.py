"""Fine-versus-parareal timing on the device path.

Mirrors the benchmark half of ``parafrac/harness.py`` (``bench_point`` /
``bench_sweep``, ``harness.py:85-123``): at ``dof = nt * m`` fine steps it
times the full-history serial solver (``run_fine_sequential``) against
``parareal_solve`` -- here both through the sm_100a library -- and records the
speedup, the iteration count and the last increment.  Timing keeps the
reference's convention (minimum over ``reps`` after ``warmup`` discarded
runs, ``time.perf_counter``, ``harness.py:65-73``); the allocation columns are
host-side ``tracemalloc`` peaks of a separate pass, as there (device memory is
owned by the library and not traced).

The truncation study of ``harness.py:126-227`` is scalar analysis of the L1
operator, not on the solver path, and is not part of the device build.
"""

from __future__ import annotations

import time
import tracemalloc
from dataclasses import dataclass

from .l1 import TimeGrids
from .problems import CONFIGS, get_problem
from .solver import parareal_solve, run_fine_sequential
from .spaces import build_operator, build_sine_operator

__all__ = ["BenchRecord", "bench_point", "bench_sweep", "make_operator"]


@dataclass(frozen=True)
class BenchRecord:
    """One sweep point; the field set of ``harness.py:46-60`` (CSV columns of ``cli bench``)."""

    dof: int
    nt: int
    m: int
    degree: int
    threads: int
    wall_fine: float
    wall_parareal: float
    speedup: float
    iterations: int
    final_diff: float
    peak_alloc_fine: int
    peak_alloc_parareal: int


def make_operator(problem, degree=None, space=None, dims=None):
    """Spatial operator for a CLI/harness run.

    ``space`` "chebyshev" is the reference's collocation operator
    (``build_operator(degree, a, b)``, ``spectral.py:74``); "sine" the
    sine-Galerkin space with ``degree`` modes per axis.  Left as ``None`` it is
    "sine" for the BASELINE problems ``cfg1``..``cfg5`` (their modes and
    dimension from ``CONFIGS`` unless ``degree`` / ``dims`` override them) and
    "chebyshev" otherwise, the reference's default.
    """
    name = getattr(problem, "name", "")
    cfg = None
    if name.startswith("cfg") and name[3:].isdigit():
        cfg = CONFIGS.get(int(name[3:]))
    if space is None:
        space = "sine" if cfg is not None else "chebyshev"
    if space == "chebyshev":
        return build_operator(16 if degree is None else int(degree), problem.a, problem.b)
    if space == "sine":
        modes = degree if degree is not None else (cfg["modes"] if cfg is not None else 16)
        d = dims if dims is not None else (cfg["dims"] if cfg is not None else 1)
        return build_sine_operator(int(modes), dims=int(d))
    raise ValueError(f"unknown space {space!r}; choices: chebyshev, sine")


class _Runner:
    """Runs one solver of a bench point: warm-up calls, timed calls
    (``time.perf_counter`` around each, the minimum kept as the reference's
    harness does, ``harness.py:65-73``) and an optional separate pass under
    ``tracemalloc`` for the host-side allocation peak (``harness.py:76-82``)."""

    def __init__(self, call):
        self.call = call
        self.last = None

    def timed(self, reps, warmup):
        for _ in range(max(0, warmup)):
            self.last = self.call()
        samples = []
        for _ in range(max(1, reps)):
            t0 = time.perf_counter()
            self.last = self.call()
            samples.append(time.perf_counter() - t0)
        return min(samples)

    def host_peak(self):
        tracemalloc.start()
        try:
            self.call()
            return int(tracemalloc.get_traced_memory()[1])
        finally:
            tracemalloc.stop()


def _grid_for(dof, m):
    """``nt * m_eff`` fine steps with ``m_eff = clip(m, 1, dof)``, ``nt = dof // m_eff``."""
    m_eff = max(1, min(int(m), int(dof)))
    return max(1, int(dof) // m_eff), m_eff


def bench_point(problem_name, dof, *, alpha=None, degree=16, m=32, tol=1e-10, k_max=20, threads=1,
                reps=3, warmup=1, measure_memory=True, space=None, dims=None):
    """Serial fine solver vs parareal at ``nt * m ~= dof`` fine steps, both on
    the device (the row schema of ``harness.py:85-117``).  ``threads`` is
    recorded and otherwise ignored (the device batches every slice)."""
    if dof < 1:
        raise ValueError("dof must be a positive integer")
    nt, m_eff = _grid_for(dof, m)
    problem = get_problem(problem_name, alpha=alpha)
    op = make_operator(problem, degree, space, dims)
    grids = TimeGrids(problem.t_final, nt, m_eff)
    serial = _Runner(lambda: run_fine_sequential(problem, op, grids))
    para = _Runner(lambda: parareal_solve(problem, op, grids, tol=tol, k_max=k_max, threads=threads))
    t_serial = serial.timed(reps, warmup)
    t_para = para.timed(reps, warmup)
    report = para.last[1]
    peaks = (serial.host_peak(), para.host_peak()) if measure_memory else (0, 0)
    return BenchRecord(dof=nt * m_eff, nt=nt, m=m_eff, degree=int(getattr(op, "degree", getattr(op, "modes", 0))),
                       threads=int(threads), wall_fine=t_serial, wall_parareal=t_para, speedup=t_serial / t_para,
                       iterations=report.iterations, final_diff=report.diffs[-1], peak_alloc_fine=peaks[0],
                       peak_alloc_parareal=peaks[1])


def bench_sweep(problem_name, dofs, **kwargs):
    """One ``bench_point`` per entry of ``dofs``, in order (``harness.py:120-123``)."""
    points = list(dofs)
    if not points:
        raise ValueError("benchmark sweep must not be empty")
    return [bench_point(problem_name, d, **kwargs) for d in points]
