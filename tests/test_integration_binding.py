"""The INTEGRATION.md binding, executed inside the UNMODIFIED reference (``-m gpu``).

INTEGRATION.md shows the ctypes stub a maintainer adds to ``parafrac``
(``parafrac/_b200.py``) and the one-line dispatch in ``_parallel_stage``
(``parareal.py:75-88``).  This test takes that code block verbatim from
INTEGRATION.md, loads it as ``parafrac._b200`` into the reference installed
under ``baseline/_ref`` (``pip install --target baseline/_ref``; it travels to
the GPU box, ``/root/reference`` does not), routes the reference's own
``parareal_solve`` through ``pf_fine_sweep`` and compares with the unpatched
reference run: same iteration count, iterates within 1e-12 relative L2."""

import os
import re
import sys
import types

import numpy as np
import pytest

from conftest import ROOT, rel_err

pytestmark = pytest.mark.gpu

REF_TARGET = os.path.join(ROOT, "baseline", "_ref")
LIB = os.path.join(ROOT, "paper_2510_11023_b200", "libparafrac_b200.so")


def _stub_source():
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    blocks = re.findall(r"```python\n(.*?)```", text, re.S)
    src = next(b for b in blocks if "parafrac/_b200.py" in b)
    assert '"libparafrac_b200.so"' in src
    return src.replace('"libparafrac_b200.so"', repr(LIB))


@pytest.fixture(scope="module")
def parafrac_with_stub():
    if not os.path.isdir(os.path.join(REF_TARGET, "parafrac")):
        pytest.skip("reference not installed under baseline/_ref (DESIGN.md §5: pip install --target)")
    import torch

    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a B200")
    sys.path.insert(0, REF_TARGET)
    try:
        import parafrac
        import parafrac.parareal as ref_parareal
    finally:
        sys.path.remove(REF_TARGET)
    assert os.path.realpath(parafrac.__file__).startswith(os.path.realpath(REF_TARGET))
    stub = types.ModuleType("parafrac._b200")
    stub.__package__ = "parafrac"
    exec(compile(_stub_source(), "INTEGRATION.md:parafrac/_b200.py", "exec"), stub.__dict__)
    sys.modules["parafrac._b200"] = stub
    return parafrac, ref_parareal, stub


def _cfg1_problem(pf):
    """BASELINE config 1 as a reference ProblemSpec (numpy callbacks), as
    tests/golden/make_golden.py builds it."""
    M = 32
    amps = np.zeros(M)
    amps[0], amps[2] = 1.0, 0.5
    k = np.arange(1, M + 1)

    def initial(x):
        return np.sin(np.pi * np.multiply.outer(np.asarray(x, dtype=float), k)) @ amps

    return pf.ProblemSpec(0.0, 1.0, 1.0, 0.5, lambda x, t, u: 1.0 + u**2 / (1.0 + u**2),
                          lambda x, t, u: np.sin(np.pi * x) * np.cos(u), initial, name="cfg1")


@pytest.mark.parametrize("case", ["paper42", "cfg1"])
def test_reference_parareal_through_the_binding(parafrac_with_stub, case, monkeypatch):
    pf, ref_parareal, stub = parafrac_with_stub
    if case == "paper42":
        prob, op, grids = pf.get_problem("paper42"), pf.build_operator(16, 0.0, 1.0), pf.TimeGrids(1.0, 16, 4)
    else:
        prob, op, grids = _cfg1_problem(pf), pf.build_operator(33, 0.0, 1.0), pf.TimeGrids(1.0, 8, 64)
    want_it, want_rep = pf.parareal_solve(prob, op, grids, tol=1e-12, k_max=grids.nt + 1)
    calls = []

    def dispatched(u_nodes, lo, hi, op_, grids_, problem_):
        calls.append((lo, hi))
        return stub.fine_sweep_intervals(u_nodes, lo, hi, op_, grids_, problem_)

    monkeypatch.setattr(ref_parareal, "fine_sweep_intervals", dispatched)
    got_it, got_rep = pf.parareal_solve(prob, op, grids, tol=1e-12, k_max=grids.nt + 1)
    assert calls and calls[0] == (0, grids.nt)  # every sweep went through the C-ABI
    assert got_rep.iterations == want_rep.iterations
    assert got_rep.stop_reason == want_rep.stop_reason
    assert rel_err(got_it.states, want_it.states) <= 1e-12
    assert rel_err(got_it.fine_endpoints, want_it.fine_endpoints) <= 1e-12
    # the binding's error path: an argument error of the reference raises ValueError
    with pytest.raises(ValueError):
        stub.fine_sweep_intervals(want_it.states, 0, grids.nt + 5, op, grids, prob)
