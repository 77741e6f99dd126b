"""Problem data for the oracle — TEST INFRASTRUCTURE ONLY.

Builtins restate ``pkg/src/parafrac/problems.py:81-133``; ``config(i)``
restates ``BASELINE.json`` configs 1-5 with the RNG convention recorded in
SURVEY.md §8(d):

* 1-D coefficients of ``sin(k pi x)``: ``a = default_rng(seed).standard_normal(M) * k**-p``;
  the orthonormal-basis coefficients are ``a / sqrt(2)``;
* 2-D: ``standard_normal((M, M)) * (k1^2 + k2^2)**-1.5`` for
  ``sin(k1 pi x) sin(k2 pi y)``, orthonormal coefficients ``a / 2``;
* "scaled to max|u0| = 1" is the max over the ``Q = 2M`` quadrature midpoints.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np


@dataclass(frozen=True)
class Problem:
    a: float
    b: float
    t_final: float
    alpha: float
    diffusion: Callable
    source: Callable
    initial: Callable
    name: str = "custom"
    initial_coefficients: Optional[Callable] = None


# reference builtins (problems.py:81-133)
def paper42():
    return Problem(0.0, 1.0, 1.0, 0.5, lambda x, t, u: 1.0 + u,
                   lambda x, t, u: np.sin(np.pi * x) * np.exp(-t),
                   lambda x: x**4 * (1.0 - x) ** 4, "paper42")


def linear_heat():
    return Problem(0.0, 1.0, 1.0, 0.5, lambda x, t, u: 1.0,
                   lambda x, t, u: np.sin(np.pi * x) * np.exp(-t),
                   lambda x: np.sin(np.pi * x), "linear-heat")


def constant_d():
    return Problem(0.0, 1.0, 1.0, 0.5, lambda x, t, u: 1.0, lambda x, t, u: 0.0,
                   lambda x: x**4 * (1.0 - x) ** 4, "constant-D")


def zero():
    return Problem(0.0, 1.0, 1.0, 0.5, lambda x, t, u: 1.0 + u, lambda x, t, u: 0.0,
                   lambda x: np.zeros_like(np.asarray(x, dtype=float)), "zero")


BUILTINS = {"paper42": paper42, "linear-heat": linear_heat, "constant-D": constant_d,
            "zero": zero}


def _sine_series(a):
    a = np.asarray(a, dtype=float)
    k = np.arange(1, a.size + 1)

    def u0(x):
        x = np.asarray(x, dtype=float)
        return np.sin(np.pi * np.multiply.outer(x, k)) @ a

    return u0


def coeffs_1d(M, seed, p, scale_to_one=False):
    """Sine-series amplitudes ``a_k`` of ``sin(k pi x)`` (length M)."""
    k = np.arange(1, M + 1, dtype=float)
    a = np.random.default_rng(seed).standard_normal(M) * k ** (-p)
    if scale_to_one:
        Q = 2 * M
        x = (np.arange(Q) + 0.5) / Q
        a = a / np.abs(np.sin(np.pi * np.outer(x, k)) @ a).max()
    return a


def coeffs_2d(M, seed):
    k = np.arange(1, M + 1, dtype=float)
    return np.random.default_rng(seed).standard_normal((M, M)) * (k[:, None] ** 2 + k[None, :] ** 2) ** -1.5


def _d12(x, t, u):
    return 1.0 + u**2 / (1.0 + u**2)


def _f12(x, t, u):
    return np.sin(np.pi * x) * np.cos(u)


def _d3(x, t, u):
    return 1.5 + 0.5 * np.tanh(u)


def _f3(x, t, u):
    return -u + 0.1 * np.sin(2.0 * np.pi * x)


def _d45(x, t, u):
    return (1.0 + 0.5 * x[0]) * (1.0 + 0.5 * np.sin(u) ** 2)


def _f45(x, t, u):
    return u * (1.0 - u**2) / (1.0 + u**2)


CONFIG_GRIDS = {  # (modes, P, m, alpha, T, tol)
    1: (32, 8, 64, 0.5, 1.0, 1e-12),
    2: (64, 16, 256, 1.0, 1.0, 1e-12),
    3: (512, 64, 1024, 0.3, 2.0, 1e-12),
    4: (128, 128, 256, 0.7, 1.0, 1e-12),
    5: (256, 512, 128, 0.5, 1.0, 1e-12),
}


def config(i, modes=None):
    """BASELINE.json config ``i`` (1-based) as a problem; ``modes`` overrides M
    for reduced-size parity runs (the random coefficients are then drawn at
    the reduced M)."""
    M0, _, _, alpha, T, _ = CONFIG_GRIDS[i]
    M = M0 if modes is None else int(modes)
    if i == 1:
        a = np.zeros(M)
        a[0] = 1.0
        if M >= 3:
            a[2] = 0.5
        return Problem(0.0, 1.0, T, alpha, _d12, _f12, _sine_series(a), "cfg1",
                       lambda MM, a=a: a[:MM] / math.sqrt(2.0))
    if i == 2:
        a = coeffs_1d(M, 1, 3.0)
        return Problem(0.0, 1.0, T, alpha, _d12, _f12, _sine_series(a), "cfg2",
                       lambda MM, a=a: a[:MM] / math.sqrt(2.0))
    if i == 3:
        a = coeffs_1d(M, 2, 2.5, scale_to_one=True)
        return Problem(0.0, 1.0, T, alpha, _d3, _f3, _sine_series(a), "cfg3",
                       lambda MM, a=a: a[:MM] / math.sqrt(2.0))
    seed = 3 if i == 4 else 4
    a2 = coeffs_2d(M, seed)
    return Problem(0.0, 1.0, T, alpha, _d45, _f45, None, f"cfg{i}",
                   lambda MM, a2=a2: a2[:MM, :MM] / 2.0)
