"""The drop-in boundary without a GPU: the C-ABI library loads and exports
every symbol include/parafrac_b200.h declares, the ctypes layouts match the
header (probed with gcc), host-side tables and problem registry follow the
reference, and compute entry points fail loudly when no B200 is present."""

import ctypes as C
import os
import re
import subprocess
import tempfile

import numpy as np
import pytest

import paper_2510_11023_b200 as pfb
from paper_2510_11023_b200 import _lib
from paper_2510_11023_b200.parallel import block_bounds

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "parafrac_b200.h")


def header_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\**(pf_\w+)\s*\(", text, re.M)))


def test_library_exports_every_declared_symbol():
    names = header_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(_lib.lib, n), n
        assert n in _lib.SIGNATURES, n
    assert _lib.lib.pf_version().startswith(b"parafrac_b200")


def test_ctypes_layouts_match_header():
    structs = ["pf_problem", "pf_grid", "pf_space", "pf_weights", "pf_error", "pf_stats"]
    src = '#include <stdio.h>\n#include <stddef.h>\n#include "parafrac_b200.h"\nint main(){\n'
    for s in structs:
        src += f'printf("{s} %zu\\n", sizeof({s}));\n'
    src += 'printf("off_error_message %zu\\n", offsetof(pf_error, message));\n'
    src += 'printf("off_space_pcg %zu\\n", offsetof(pf_space, pcg_tol));\nreturn 0;}\n'
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "probe.c")
        exe = os.path.join(d, "probe")
        open(c, "w").write(src)
        subprocess.run(["gcc", "-I", os.path.dirname(HEADER), c, "-o", exe], check=True)
        out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout.split()
    got = dict(zip(out[0::2], map(int, out[1::2])))
    for s in structs:
        assert got[s] == C.sizeof(getattr(_lib, s)), s
    assert got["off_error_message"] == _lib.pf_error.message.offset
    assert got["off_space_pcg"] == _lib.pf_space.pcg_tol.offset


def test_host_weights_match_oracle():
    import oracle

    for alpha in (0.3, 0.5, 1.0):
        a = pfb.weights_for(alpha)
        b = oracle.weights_for(alpha)
        np.testing.assert_array_equal(a.on_grid(1, 300), b.on_grid(1, 300))
        np.testing.assert_array_equal(a.on_grid(64, 3000), b.on_grid(64, 3000))
    assert pfb.gamma_2_minus(0.5) == oracle.gamma_2_minus(0.5)


def test_block_bounds_contract():
    for count in (1, 5, 8, 17, 64):
        for parts in (1, 2, 3, 8, 32):
            b = block_bounds(count, parts)
            assert b[0][0] == 0 and b[-1][1] == count and len(b) == min(parts, count)
            assert all(x[1] == y[0] and x[1] > x[0] for x, y in zip(b, b[1:]))


def _functor_numpy(fid, p, x, t, u):
    """numpy restatement of the PF_FN_* formulas documented in the header."""
    if fid == 1:
        return p[0] + p[1] * u, p[2] * u + p[3] * (np.sin(np.pi * x) * np.exp(-t))
    if fid == 2:
        return 1.0 + u**2 / (1.0 + u**2), np.sin(np.pi * x) * np.cos(u)
    if fid == 3:
        return 1.5 + 0.5 * np.tanh(u), -u + 0.1 * np.sin(2.0 * np.pi * x)
    if fid == 4:
        return (1.0 + 0.5 * x) * (1.0 + 0.5 * np.sin(u) ** 2), u * (1.0 - u**2) / (1.0 + u**2)
    raise AssertionError(fid)


@pytest.mark.parametrize("name", ["paper42", "linear-heat", "constant-D", "zero", "cfg1", "cfg2", "cfg3"])
def test_device_functor_matches_callbacks(name):
    prob = pfb.get_problem(name)
    fid, p = prob.device_functor()
    rng = np.random.default_rng(3)
    x, t, u = rng.random(50), 0.37, rng.standard_normal(50)
    d, f = _functor_numpy(fid, p, x, t, u)
    np.testing.assert_allclose(np.broadcast_to(prob.diffusion(x, t, u), x.shape), d, rtol=1e-15, atol=0)
    np.testing.assert_allclose(np.broadcast_to(prob.source(x, t, u), x.shape), f, rtol=1e-15, atol=1e-300)


def test_config_coefficients_and_rng_convention():
    import oracle.problems as OP

    for i in (1, 2, 3):
        a = pfb.config_problem(i).initial_coefficients(pfb.problems.CONFIGS[i]["modes"])
        b = OP.config(i).initial_coefficients(pfb.problems.CONFIGS[i]["modes"])
        np.testing.assert_array_equal(a, b)
    c3 = pfb.config_problem(3)
    op = pfb.build_sine_operator(512)
    u = (np.sqrt(2.0) * np.sin(np.pi * np.outer(op.quadrature_points, np.arange(1, 513)))) @ c3.initial_coefficients(512)
    assert abs(np.abs(u).max() - 1.0) <= 1e-12


def test_problem_validation():
    with pytest.raises(ValueError):
        pfb.get_problem("nope")
    with pytest.raises(ValueError):
        pfb.ProblemSpec(0.0, 1.0, 1.0, 0.5, lambda x, t, u: 1.0, lambda x, t, u: 0.0, lambda x: 1.0 + 0 * x)
    custom = pfb.ProblemSpec(0.0, 1.0, 1.0, 0.5, lambda x, t, u: 1.0, lambda x, t, u: 0.0,
                             lambda x: np.sin(np.pi * np.asarray(x)))
    with pytest.raises(ValueError, match="device coefficient functor"):
        custom.device_functor()
    with pytest.raises(ValueError):
        pfb.build_sine_operator(12)
    assert pfb.get_problem("paper42", alpha=0.7).alpha == 0.7


def test_initial_state_projection_exact_for_bandlimited():
    prob = pfb.get_problem("linear-heat")  # u0 = sin(pi x)
    c = pfb.initial_state(prob, pfb.build_sine_operator(16))
    want = np.zeros(16)
    want[0] = 1.0 / np.sqrt(2.0)
    np.testing.assert_allclose(c, want, atol=1e-15)


def test_chebyshev_operator_matches_oracle():
    import oracle

    a = pfb.build_operator(17, 0.0, 1.0)
    b = oracle.build_operator(17, 0.0, 1.0)
    np.testing.assert_array_equal(a.d1, b.d1)
    np.testing.assert_array_equal(a.quad_weights, b.quad_weights)
    np.testing.assert_array_equal(a.nodes, b.nodes)


def test_compute_fails_loudly_without_gpu():
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    prob = pfb.get_problem("paper42")
    op = pfb.build_operator(8, 0.0, 1.0)
    with pytest.raises(pfb.DeviceError):
        pfb.run_coarse(prob, op, pfb.TimeGrids(1.0, 4, 2))


def test_reference_argument_errors_without_gpu():
    prob = pfb.get_problem("paper42")
    op = pfb.build_operator(8, 0.0, 1.0)
    g = pfb.TimeGrids(1.0, 4, 2)
    with pytest.raises(ValueError):
        pfb.parareal_solve(prob, op, g, tol=0.0)
    with pytest.raises(ValueError):
        pfb.parareal_solve(prob, op, g, k_max=0)
    with pytest.raises(ValueError):
        pfb.parareal_solve(prob, op, g, threads=0)
    with pytest.raises(ValueError):
        pfb.fine_sweep_intervals(np.zeros((3, 7)), 0, 3, op, g, prob)
    with pytest.raises(ValueError):
        pfb.coarse_step(np.empty((0, 7)), op, g, prob)
