"""Spatial operators the device path accepts as ``op``.

* ``build_operator(degree, a, b)`` — the reference's Chebyshev-Lobatto
  collocation operator (``spectral.py:74-103``), built with the reference's
  exact numpy expressions so the arrays handed to the device are bit-identical
  to the reference's.  On the device it runs the dense bridge kernel
  (assembly + LU in shared memory).
* ``build_sine_operator(modes)`` — the sine spectral-Galerkin basis
  ``sqrt(2) sin(k pi x)``, ``k = 1..M``, with ``Q = 2M`` midpoint quadrature
  (SURVEY.md §8.0).  The device applies it matrix-free through FFT-based
  DCT-II/III pairs; nothing dense is formed.

Both expose ``interior_size`` / ``size`` (the state length), ``l2_norm`` and
``initial_state`` exactly as the reference (``spectral.py:130-136``,
``stepping.py:51-54``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

__all__ = ["ChebyshevOperator", "SineOperator", "build_operator", "build_sine_operator",
           "clenshaw_curtis_weights", "initial_state", "l2_norm"]

SPACE_CHEB1D, SPACE_SINE1D, SPACE_SINE2D = 1, 2, 3


def clenshaw_curtis_weights(degree):
    """Quadrature weights on the ``degree + 1`` Lobatto nodes (``spectral.py:27-45``)."""
    if degree < 1:
        raise ValueError("need at least two quadrature nodes")
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


@dataclass(frozen=True, eq=False)
class ChebyshevOperator:
    """Collocation operator on ``[a, b]`` (``spectral.py:48-71``)."""

    degree: int
    a: float
    b: float
    nodes: np.ndarray
    d1: np.ndarray
    d2: np.ndarray
    quad_weights: np.ndarray
    kind: int = SPACE_CHEB1D

    @property
    def interior_size(self):
        return self.degree - 1

    size = interior_size

    @property
    def interior_nodes(self):
        return self.nodes[1:-1]


def build_operator(degree, a, b):
    """``spectral.build_operator`` (``spectral.py:74-103``)."""
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
    d2 = d1 @ d1
    nodes = 0.5 * (a + b) + 0.5 * (b - a) * xi
    qw = clenshaw_curtis_weights(degree) * (0.5 * (b - a))
    for arr in (nodes, d1, d2, qw):
        arr.setflags(write=False)
    return ChebyshevOperator(degree=degree, a=float(a), b=float(b), nodes=nodes, d1=d1, d2=d2,
                             quad_weights=qw)


@dataclass(frozen=True, eq=False)
class SineOperator:
    """Sine spectral-Galerkin space on (0, 1): ``M`` modes per axis, ``dims`` 1 or 2.

    ``pcg_tol`` is the relative-residual tolerance of the device PCG
    (``||r||_2 <= pcg_tol ||rhs||_2``); ``pcg_maxit`` caps its iterations.
    """

    modes: int
    dims: int = 1
    pcg_tol: float = 1e-14
    pcg_maxit: int = 500

    def __post_init__(self):
        if self.modes < 1 or self.modes & (self.modes - 1):
            raise ValueError("sine modes must be a power of two")
        if self.dims not in (1, 2):
            raise ValueError("dims must be 1 or 2")

    @property
    def kind(self):
        return SPACE_SINE1D if self.dims == 1 else SPACE_SINE2D

    @property
    def a(self):
        return 0.0

    @property
    def b(self):
        return 1.0

    @property
    def Q(self):
        return 2 * self.modes

    @property
    def interior_size(self):
        return self.modes ** self.dims

    size = interior_size

    @property
    def quadrature_points(self):
        return (np.arange(self.Q) + 0.5) / self.Q


def build_sine_operator(modes, dims=1, pcg_tol=None, pcg_maxit=500):
    tol = (1e-14 if dims == 1 else 1e-13) if pcg_tol is None else pcg_tol
    return SineOperator(int(modes), int(dims), float(tol), int(pcg_maxit))


def initial_state(problem, op):
    """State at t=0 (``stepping.py:51-54``).

    Collocation: ``initial`` at the interior nodes.  Sine: the problem's
    coefficient generator when it has one, else the quadrature projection
    ``c_k = sum_q w_q u0(x_q) sqrt(2) sin(k pi x_q)`` (exact for band-limited u0).
    """
    if isinstance(op, ChebyshevOperator):
        u0 = np.asarray(problem.initial(op.interior_nodes), dtype=float)
        return np.broadcast_to(u0, (op.interior_size,)).astype(float, copy=True)
    gen = getattr(problem, "initial_coefficients", None)
    if gen is not None:
        c = np.asarray(gen(op.modes), dtype=float)
        return np.ascontiguousarray(c.reshape(-1))
    x = op.quadrature_points
    k = np.arange(1, op.modes + 1)
    S = math.sqrt(2.0) * np.sin(np.pi * np.outer(x, k))
    if op.dims == 1:
        return (np.asarray(problem.initial(x), dtype=float) / op.Q) @ S
    X1, X2 = np.meshgrid(x, x, indexing="ij")
    U0 = np.asarray(problem.initial((X1, X2)), dtype=float)
    return (S.T @ (U0 / op.Q**2) @ S).reshape(-1)


def l2_norm(op, values):
    """Discrete L2 norm: Clenshaw-Curtis interior weights (``spectral.py:130-136``)
    for collocation, the coefficient Euclidean norm (Parseval) for sine spaces."""
    v = np.asarray(values, dtype=float)
    if isinstance(op, ChebyshevOperator):
        return math.sqrt(float(np.dot(op.quad_weights[1:-1], np.square(v))))
    return math.sqrt(float(np.dot(v.ravel(), v.ravel())))
