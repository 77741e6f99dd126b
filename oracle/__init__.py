"""CPU oracle for the parareal fine-propagator path — TEST INFRASTRUCTURE ONLY.

This package is a numpy restatement of the reference ``parafrac`` algorithm
(``pkg/src/parafrac/{l1,stepping,parareal,spectral}.py``) with a pluggable
spatial operator:

* ``ChebyshevSpace`` — the reference's own collocation operator
  (``spectral.py:74-136``); with it the restatement reproduces the imported
  reference bit for bit on this host (pinned by ``tests/test_oracle_pin.py``
  and the fixtures in ``tests/golden/``).
* ``Sine1D`` / ``Sine2D`` — the sine spectral-Galerkin operator the
  BASELINE configs name.  Not present in the reference;
  the time-stepping algebra around it is the reference's unchanged.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package, and only
as the checker or the timed CPU baseline.  The product path
(``paper_2510_11023_b200``) never imports it and has no CPU fallback.
"""

from .weights import (
    FractionalWeights,
    TimeGrids,
    gamma_2_minus,
    history_weights,
    l1_weight,
    weights_for,
)
from .spaces import ChebyshevSpace, Sine1D, Sine2D, build_operator
from .stepping import (
    chain_fine,
    coarse_contribution,
    coarse_step,
    fine_propagate,
    fine_sweep_intervals,
    run_coarse,
    run_fine_sequential,
)
from .parareal import block_bounds, exactness_check, parareal_solve, solve
from . import problems

__all__ = [
    "ChebyshevSpace",
    "FractionalWeights",
    "Sine1D",
    "Sine2D",
    "TimeGrids",
    "block_bounds",
    "build_operator",
    "chain_fine",
    "coarse_contribution",
    "coarse_step",
    "exactness_check",
    "fine_propagate",
    "fine_sweep_intervals",
    "gamma_2_minus",
    "history_weights",
    "l1_weight",
    "parareal_solve",
    "problems",
    "run_coarse",
    "run_fine_sequential",
    "solve",
    "weights_for",
]
