"""B200-native parareal-L1-spectral solver (drop-in for ``parafrac``'s solver path).

Public surface mirrors ``parafrac/__init__.py:9-84`` for the solver subset:
``parareal_solve``, ``fine_sweep_intervals`` (the hot path), ``coarse_step``,
``run_coarse``, ``fine_propagate``, ``chain_fine``, ``run_fine_sequential``,
``exactness_check``, problems, grids, operators and exceptions.  Compute runs
in ``libparafrac_b200.so`` (hand-written sm_100a CUDA behind a C-ABI); there is
no CPU fallback.  ``parallel`` holds the multi-GPU (one process per GPU)
driver.
"""

from .errors import CoefficientError, DeviceError, DivergenceError, ParafracError, SolverFailure
from .l1 import FractionalWeights, TimeGrids, gamma_2_minus, l1_weight, weights_for
from .problems import ProblemSpec, config_problem, get_problem, registry_names
from .spaces import (ChebyshevOperator, SineOperator, build_operator, build_sine_operator,
                     initial_state, l2_norm)
from .solver import (PararealIterate, PararealReport, chain_fine, coarse_step, exactness_check,
                     fine_propagate, fine_sweep_intervals, parareal_solve, run_coarse,
                     run_fine_sequential)

__version__ = "0.1.0"

__all__ = [
    "ChebyshevOperator", "CoefficientError", "DeviceError", "DivergenceError", "FractionalWeights",
    "ParafracError", "PararealIterate", "PararealReport", "ProblemSpec", "SineOperator",
    "SolverFailure", "TimeGrids", "build_operator", "build_sine_operator", "chain_fine",
    "coarse_step", "config_problem", "exactness_check", "fine_propagate", "fine_sweep_intervals",
    "gamma_2_minus", "get_problem", "initial_state", "l1_weight", "l2_norm", "parareal_solve",
    "registry_names", "run_coarse", "run_fine_sequential", "weights_for",
]
