"""L1 weights and nested time grids — host side of the weight tables.

The device never evaluates ``(x+1)^e - x^e`` itself on this path: the host
computes the tables with the reference's exact numpy expressions
(``l1.py:127-166``) and uploads them, so device results follow the same
rounding of the catastrophically cancelling weights that the
reference sees on this host.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from functools import lru_cache

import numpy as np

__all__ = ["FractionalWeights", "TimeGrids", "gamma_2_minus", "l1_weight", "weights_for"]


def _check_alpha(alpha):
    if not 0.0 < alpha <= 1.0:
        raise ValueError(f"fractional order must lie in (0, 1], got {alpha}")


def gamma_2_minus(alpha):
    """``Gamma(2 - alpha)`` on the log scale (``l1.py:40-42``)."""
    return math.exp(math.lgamma(2.0 - alpha))


def l1_weight(x, alpha):
    """``b_x = (x+1)^(1-alpha) - x^(1-alpha)``; exact zeros at alpha=1 (``l1.py:45-58``)."""
    if x < 0:
        raise ValueError(f"weight index must be nonnegative, got {x}")
    _check_alpha(alpha)
    if alpha == 1.0:
        return 1.0 if x == 0.0 else 0.0
    e = 1.0 - alpha
    return (x + 1.0) ** e - x ** e


@dataclass(frozen=True)
class TimeGrids:
    """``nt`` coarse intervals of ``m`` fine steps each (``l1.py:61-96``)."""

    t_final: float
    nt: int
    m: int

    def __post_init__(self):
        if not self.t_final > 0:
            raise ValueError(f"final time must be positive, got {self.t_final}")
        if self.nt < 1 or self.m < 1:
            raise ValueError("grid counts nt and m must be positive integers")

    @property
    def dT(self):
        return self.t_final / self.nt

    @property
    def dt(self):
        return self.dT / self.m

    @property
    def total_fine(self):
        return self.nt * self.m

    def coarse_node(self, n):
        return n * self.dT

    def fine_node(self, n, r):
        return n * self.dT + r * self.dt


class FractionalWeights:
    """Memoised weight grids ``b_{q/denom}`` for one order (``l1.py:99-166``)."""

    __slots__ = ("alpha", "_grids", "_rows")

    def __init__(self, alpha):
        _check_alpha(alpha)
        self.alpha = float(alpha)
        self._grids = {}
        self._rows = {}

    def value(self, x):
        return l1_weight(x, self.alpha)

    def on_grid(self, denom, count):
        if denom < 1 or count < 1:
            raise ValueError("denominator and count must be positive")
        arr = self._grids.get(denom)
        if arr is None or arr.shape[0] < count:
            size = max(count, 64, 0 if arr is None else 2 * arr.shape[0])
            x = np.arange(size, dtype=float) / denom
            if self.alpha == 1.0:
                new = np.zeros(size)
                new[0] = 1.0
            else:
                e = 1.0 - self.alpha
                new = (x + 1.0) ** e - x ** e
            new.setflags(write=False)
            self._grids[denom] = new
            arr = new
        return arr[:count]

    def fine_rows(self, m):
        rows = self._rows.get(m)
        if rows is None:
            b = self.on_grid(1, m + 1)
            built = []
            for r in range(1, m + 1):
                w = np.empty(r)
                w[0] = b[r - 1]
                if r > 1:
                    j = np.arange(1, r)
                    w[1:] = b[r - j - 1] - b[r - j]
                w.setflags(write=False)
                built.append(w)
            rows = tuple(built)
            self._rows[m] = rows
        return rows


@lru_cache(maxsize=16)
def weights_for(alpha):
    """Process-wide weight table per order (``l1.py:169-172``)."""
    return FractionalWeights(alpha)
