"""Sine spectral-Galerkin oracle: operator identities, the
PCG the device runs vs the direct solve, the reference's structural
properties restated for the sine space, and the cross-discretisation check
against the reference's own Chebyshev run of config 1."""

import math

import numpy as np
import pytest

import oracle
from oracle import problems as P

from conftest import rel_err, sine_u


def test_basis_orthonormal_and_operator_spd():
    sp = oracle.Sine1D(16)
    np.testing.assert_allclose(sp.w * sp.S.T @ sp.S, np.eye(16), atol=1e-14)
    d = sp.w * (1.0 + 0.5 * np.sin(3 * sp.x) ** 2)
    K = (sp.Sp.T * d) @ sp.Sp
    np.testing.assert_allclose(K, K.T, atol=1e-12)
    assert np.linalg.eigvalsh(K).min() > 0
    v = np.random.default_rng(0).standard_normal(16)
    np.testing.assert_allclose(sp.apply_k(d, v), K @ v, rtol=1e-12, atol=1e-12)


def test_constant_coefficient_is_diagonal():
    """D = 1: K = diag(pi^2 k^2) exactly up to round-off (quadrature exact)."""
    sp = oracle.Sine1D(32)
    K = (sp.Sp.T * (sp.w * np.ones(sp.Q))) @ sp.Sp
    np.testing.assert_allclose(K, np.diag((np.pi * sp.k) ** 2), atol=1e-9)


def test_pcg_matches_direct():
    prob = P.config(3, modes=64)
    g = oracle.TimeGrids(2.0, 4, 8)
    direct = oracle.Sine1D(64)
    pcg = oracle.Sine1D(64, solver="pcg", pcg_tol=1e-14)
    U = oracle.run_coarse(prob, direct, g)
    a = oracle.fine_sweep_intervals(U, 0, 4, direct, g, prob)
    b = oracle.fine_sweep_intervals(U, 0, 4, pcg, g, prob)
    assert rel_err(b, a) <= 1e-13
    assert 1 <= np.mean(pcg.pcg_iterations) <= 30


def test_m1_fine_equals_coarse():
    prob = P.config(1, modes=16)
    sp = oracle.Sine1D(16)
    g = oracle.TimeGrids(1.0, 12, 1)
    traj = oracle.run_coarse(prob, sp, g)
    for n in range(12):
        end, _ = oracle.fine_propagate(traj[n], traj[: n + 1], sp, g, prob)
        assert np.abs(end - traj[n + 1]).max() <= 1e-12


def test_finite_termination_sine():
    prob = P.config(2, modes=16)
    sp = oracle.Sine1D(16)
    g = oracle.TimeGrids(1.0, 6, 8)
    for k in (1, 3, 6):
        assert oracle.exactness_check(prob, sp, g, k) <= 1e-10


def test_alpha_one_is_backward_euler():
    prob = P.config(2, modes=8)
    sp = oracle.Sine1D(8)
    g = oracle.TimeGrids(1.0, 4, 1)
    traj = oracle.run_coarse(prob, sp, g)
    c = traj[1]
    u = sp.S @ traj[0]
    d = sp.w * prob.diffusion(sp.x, 0.0, u)
    F = (sp.w * prob.source(sp.x, 0.0, u)) @ sp.S
    K = (sp.Sp.T * d) @ sp.Sp
    want = np.linalg.solve(np.eye(8) + g.dT * K, traj[0] + g.dT * F)
    np.testing.assert_allclose(c, want, rtol=0, atol=1e-13)


def test_config1_sine_vs_reference_chebyshev(golden):
    """Same PDE, two discretisations: the sine-Galerkin parareal solution of
    config 1 agrees with the reference's Chebyshev run (2e-13)."""
    prob = P.config(1)
    sp = oracle.Sine1D(32)
    it, rep = oracle.solve(prob, sp, oracle.TimeGrids(1.0, 8, 64), tol=1e-12, k_max=9)
    assert rep.iterations == int(golden["cheb_cfg1_iterations"])
    cheb = oracle.build_operator(33, 0.0, 1.0)
    x = cheb.interior_nodes
    u_sine = sine_u(it.states[-1], x)
    u_cheb = golden["cheb_cfg1_states"][-1]
    assert np.abs(u_sine - u_cheb).max() <= 1e-10


def test_sine2d_operator_and_pcg():
    sp = oracle.Sine2D(8, pcg_tol=1e-13)
    rng = np.random.default_rng(1)
    d = sp.w * (1.0 + 0.3 * rng.random((sp.Q, sp.Q)))
    v, w = rng.standard_normal(64), rng.standard_normal(64)
    assert abs(v @ sp.apply_k(d, w) - w @ sp.apply_k(d, v)) <= 1e-10 * abs(v @ sp.apply_k(d, v))
    K = np.column_stack([sp.apply_k(d, e) for e in np.eye(64)])
    rhs = rng.standard_normal(64)
    x = sp.solve(d[None], 1e-3, rhs[None], 0, True)[0]
    np.testing.assert_allclose(x, np.linalg.solve(np.eye(64) + 1e-3 * K, rhs), rtol=1e-11, atol=1e-12)


def test_sine2d_parareal_finite_termination():
    prob = P.config(4, modes=4)
    sp = oracle.Sine2D(4)
    g = oracle.TimeGrids(1.0, 4, 4)
    assert oracle.exactness_check(prob, sp, g, 4) <= 1e-10


def test_full_size_config3_oracle_fixture_contract():
    """tests/golden/oracle_cfg3_full.npz (make_oracle_full.py: the oracle at the
    full config-3 size, ~2 h of CPU) -- the fixture the device is held to in
    test_gpu_parity.py::test_config3_full_size_properties."""
    import os

    f = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "oracle_cfg3_full.npz"))
    assert f["states"].shape == (65, 512) and f["fine_endpoints"].shape == (64, 512)
    assert int(f["iterations"]) == 7 == len(f["diffs"])
    d = f["diffs"]
    assert np.all(d[1:] < d[:-1]) and d[-1] < 1e-12 <= d[-2]
    assert np.isfinite(f["states"]).all()
