"""L1 weights and time grids — restatement of ``pkg/src/parafrac/l1.py``.

Oracle (test infrastructure).  The formulas are kept exactly as the
reference evaluates them, including the catastrophically cancelling
``(x+1)**e - x**e`` (``l1.py:57-58,139-140``): a more accurate formula would
*deviate* from the reference.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from functools import lru_cache

import numpy as np


def _check_alpha(alpha):
    if not 0.0 < alpha <= 1.0:
        raise ValueError(f"fractional order must lie in (0, 1], got {alpha}")


def gamma_2_minus(alpha):
    """Gamma(2 - alpha) on the log scale (``l1.py:40-42``)."""
    return math.exp(math.lgamma(2.0 - alpha))


def l1_weight(x, alpha):
    """Scalar ``b_x`` with the exact alpha=1 short-circuit (``l1.py:45-58``)."""
    if x < 0:
        raise ValueError(f"weight index must be nonnegative, got {x}")
    _check_alpha(alpha)
    if alpha == 1.0:
        return 1.0 if x == 0.0 else 0.0
    e = 1.0 - alpha
    return (x + 1.0) ** e - x ** e


@dataclass(frozen=True)
class TimeGrids:
    """Nested uniform grids (``l1.py:61-96``)."""

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


class FractionalWeights:
    """Weight grids ``b_{q/denom}`` and fine rows (``l1.py:99-166``)."""

    def __init__(self, alpha):
        _check_alpha(alpha)
        self.alpha = float(alpha)
        self._grids = {}
        self._rows = {}

    def on_grid(self, denom, count):
        """``b_{q/denom}`` for ``q < count`` (``l1.py:127-144``).

        The grow-by-doubling sizing of the reference is kept because the
        arrays are evaluated elementwise, so a longer array has the same
        leading entries.
        """
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
        """``rows[r-1][0] = b_{r-1}``, ``rows[r-1][j] = b_{r-j-1}-b_{r-j}`` (``l1.py:146-166``)."""
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
                built.append(w)
            rows = tuple(built)
            self._rows[m] = rows
        return rows


@lru_cache(maxsize=16)
def weights_for(alpha):
    """Process-wide table per order (``l1.py:169-172``)."""
    return FractionalWeights(alpha)


def history_weights(b, n):
    """Telescoped coarse weights on nodes ``0..n`` (``stepping.py:78-84``)."""
    w = np.empty(n + 1)
    w[0] = b[n]
    if n > 0:
        w[1:] = (b[:n] - b[1 : n + 1])[::-1]
    return w
