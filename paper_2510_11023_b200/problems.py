"""Problem data: the reference's ``ProblemSpec`` plus a device coefficient functor.

``ProblemSpec`` keeps the reference's fields and checks (``problems.py:23-74``)
— numpy callbacks ``diffusion(x, t, u)``, ``source(x, t, u)``, ``initial(x)``
— and adds ``device = (functor_id, params)``, the sm_100a functor that
evaluates the same D and f inside the kernels (include/parafrac_b200.h
``PF_FN_*``).  Python callbacks cannot run on the device, so a problem without
a device functor is rejected by the solver (``ValueError``); there is no CPU
fallback.  ``initial`` is evaluated on the host exactly as the reference does
(``stepping.py:51-54``).

Builtins restate the reference registry (``problems.py:81-133``); ``cfg1`` ..
``cfg5`` restate BASELINE.json's configs with the RNG convention of
SURVEY.md §8(d) (coefficients of ``sin(k pi x)`` drawn as
``default_rng(seed).standard_normal(M) * k**-p``).
"""

from __future__ import annotations

import dataclasses
import math
from dataclasses import dataclass
from typing import Callable, Optional, Tuple

import numpy as np

__all__ = ["ProblemSpec", "get_problem", "registry_names", "config_problem", "CONFIGS",
           "FN_POLY", "FN_CFG12", "FN_CFG3", "FN_CFG45", "FN_NAN_AT"]

BOUNDARY_TOL = 1e-12

FN_POLY, FN_CFG12, FN_CFG3, FN_CFG45, FN_NAN_AT = 1, 2, 3, 4, 5


@dataclass(frozen=True)
class ProblemSpec:
    """Initial-boundary value problem on ``[a, b] x (0, t_final]`` (``problems.py:23-74``)."""

    a: float
    b: float
    t_final: float
    alpha: float
    diffusion: Callable
    source: Callable
    initial: Callable
    name: str = "custom"
    d_minus: Optional[float] = None
    device: Optional[Tuple[int, Tuple[float, ...]]] = None
    initial_coefficients: Optional[Callable] = None

    def __post_init__(self):
        if not self.a < self.b:
            raise ValueError(f"invalid interval [{self.a}, {self.b}]")
        if not self.t_final > 0:
            raise ValueError(f"final time must be positive, got {self.t_final}")
        if not 0.0 < self.alpha <= 1.0:
            raise ValueError(f"fractional order must lie in (0, 1], got {self.alpha}")
        if self.initial is not None:
            for endpoint in (self.a, self.b):
                if abs(float(self.initial(endpoint))) > BOUNDARY_TOL:
                    raise ValueError(
                        "initial data must vanish at the boundary "
                        f"(got {self.initial(endpoint)} at x={endpoint})"
                    )
        if self.d_minus is not None:
            self._check_coercivity()

    def _check_coercivity(self):
        if not self.d_minus > 0:
            raise ValueError("d_minus must be positive")
        x = np.linspace(self.a, self.b, 33)
        u0 = np.broadcast_to(np.asarray(self.initial(x), dtype=float), x.shape)
        probes_u = {0.0, float(u0.min()), float(u0.max())}
        for t in np.linspace(0.0, self.t_final, 5):
            for uval in probes_u:
                d = np.broadcast_to(
                    np.asarray(self.diffusion(x, float(t), np.full_like(x, uval)), dtype=float), x.shape)
                if (d < self.d_minus).any():
                    raise ValueError(f"diffusion drops below d_minus={self.d_minus} on probe points")

    def device_functor(self):
        """``(functor_id, params[6])`` for the C-ABI, or ValueError."""
        if self.device is None:
            raise ValueError(
                f"problem {self.name!r} has no device coefficient functor; Python callbacks cannot run "
                "on the GPU path (use get_problem(...) or ProblemSpec(..., device=(FN_*, params)))")
        fid, params = self.device
        p = list(params) + [0.0] * (6 - len(params))
        return int(fid), tuple(float(v) for v in p[:6])


# ---- builtin coefficient functions (problems.py:81-104) -------------------

def one_plus_u(x, t, u):
    return 1.0 + u


def unit_coefficient(x, t, u):
    return 1.0


def decaying_sine_source(x, t, u):
    return np.sin(np.pi * x) * np.exp(-t)


def zero_source(x, t, u):
    return 0.0


def quartic_bump(x):
    return x**4 * (1.0 - x) ** 4


def sine_bump(x):
    return np.sin(np.pi * x)


def zero_initial(x):
    return np.zeros_like(np.asarray(x, dtype=float))


def _paper42():
    return ProblemSpec(0.0, 1.0, 1.0, 0.5, one_plus_u, decaying_sine_source, quartic_bump,
                       name="paper42", d_minus=0.5, device=(FN_POLY, (1.0, 1.0, 0.0, 1.0)))


def _linear_heat():
    return ProblemSpec(0.0, 1.0, 1.0, 0.5, unit_coefficient, decaying_sine_source, sine_bump,
                       name="linear-heat", d_minus=0.9, device=(FN_POLY, (1.0, 0.0, 0.0, 1.0)))


def _constant_d():
    return ProblemSpec(0.0, 1.0, 1.0, 0.5, unit_coefficient, zero_source, quartic_bump,
                       name="constant-D", d_minus=0.9, device=(FN_POLY, (1.0, 0.0, 0.0, 0.0)))


def _zero():
    return ProblemSpec(0.0, 1.0, 1.0, 0.5, one_plus_u, zero_source, zero_initial, name="zero",
                       device=(FN_POLY, (1.0, 1.0, 0.0, 0.0)))


# ---- BASELINE.json configs -------------------------------------------------

def _d12(x, t, u):
    return 1.0 + u**2 / (1.0 + u**2)


def _f12(x, t, u):
    return np.sin(np.pi * x) * np.cos(u)


def _d3(x, t, u):
    return 1.5 + 0.5 * np.tanh(u)


def _f3(x, t, u):
    return -u + 0.1 * np.sin(2.0 * np.pi * x)


def _d45(x, t, u):
    x1 = x[0] if isinstance(x, tuple) else x
    return (1.0 + 0.5 * x1) * (1.0 + 0.5 * np.sin(u) ** 2)


def _f45(x, t, u):
    return u * (1.0 - u**2) / (1.0 + u**2)


# (modes, slices P, fine steps m, alpha, T, parareal tol, dims)
CONFIGS = {
    1: dict(modes=32, nt=8, m=64, alpha=0.5, t_final=1.0, tol=1e-12, dims=1),
    2: dict(modes=64, nt=16, m=256, alpha=1.0, t_final=1.0, tol=1e-12, dims=1),
    3: dict(modes=512, nt=64, m=1024, alpha=0.3, t_final=2.0, tol=1e-12, dims=1),
    4: dict(modes=128, nt=128, m=256, alpha=0.7, t_final=1.0, tol=1e-12, dims=2, pcg_tol=1e-13),
    5: dict(modes=256, nt=512, m=128, alpha=0.5, t_final=1.0, tol=1e-12, dims=2),
}


def _sine_series(amps):
    amps = np.asarray(amps, dtype=float)
    k = np.arange(1, amps.size + 1)

    def initial(x):
        x = np.asarray(x, dtype=float)
        return np.sin(np.pi * np.multiply.outer(x, k)) @ amps

    return initial


def _amplitudes_1d(M, seed, p, scale_to_one):
    k = np.arange(1, M + 1, dtype=float)
    a = np.random.default_rng(seed).standard_normal(M) * k ** (-p)
    if scale_to_one:
        Q = 2 * M
        x = (np.arange(Q) + 0.5) / Q
        a = a / np.abs(np.sin(np.pi * np.outer(x, k)) @ a).max()
    return a


def config_problem(i, modes=None):
    """BASELINE config ``i`` as a problem (``modes`` overrides M for reduced runs)."""
    cfg = CONFIGS[i]
    M = cfg["modes"] if modes is None else int(modes)
    alpha, T = cfg["alpha"], cfg["t_final"]
    if i in (1, 2, 3):
        if i == 1:
            amps = np.zeros(M)
            amps[0] = 1.0
            if M >= 3:
                amps[2] = 0.5
            d, f, dev = _d12, _f12, (FN_CFG12, ())
        elif i == 2:
            amps = _amplitudes_1d(M, 1, 3.0, False)
            d, f, dev = _d12, _f12, (FN_CFG12, ())
        else:
            amps = _amplitudes_1d(M, 2, 2.5, True)
            d, f, dev = _d3, _f3, (FN_CFG3, ())
        coeffs = amps / math.sqrt(2.0)
        return ProblemSpec(0.0, 1.0, T, alpha, d, f, _sine_series(amps), name=f"cfg{i}",
                           device=dev, initial_coefficients=lambda MM, c=coeffs: c[:MM].copy())
    k = np.arange(1, M + 1, dtype=float)
    seed = 3 if i == 4 else 4
    amps2 = np.random.default_rng(seed).standard_normal((M, M)) * (k[:, None] ** 2 + k[None, :] ** 2) ** -1.5
    coeffs2 = amps2 / 2.0
    return ProblemSpec(0.0, 1.0, T, alpha, _d45, _f45, None, name=f"cfg{i}",
                       device=(FN_CFG45, ()), initial_coefficients=lambda MM, c=coeffs2: c[:MM, :MM].copy())


_REGISTRY = {
    "paper42": _paper42,
    "linear-heat": _linear_heat,
    "constant-D": _constant_d,
    "zero": _zero,
    "cfg1": lambda: config_problem(1),
    "cfg2": lambda: config_problem(2),
    "cfg3": lambda: config_problem(3),
    "cfg4": lambda: config_problem(4),
    "cfg5": lambda: config_problem(5),
}


def registry_names():
    return sorted(_REGISTRY)


def get_problem(name, alpha=None, t_final=None):
    """Builtin problem with optional order / horizon overrides (``problems.py:140-156``)."""
    try:
        factory = _REGISTRY[name]
    except KeyError:
        raise ValueError(f"unknown problem {name!r}; builtins: {', '.join(registry_names())}") from None
    problem = factory()
    overrides = {}
    if alpha is not None:
        overrides["alpha"] = float(alpha)
    if t_final is not None:
        overrides["t_final"] = float(t_final)
    if overrides:
        problem = dataclasses.replace(problem, **overrides)
    return problem
