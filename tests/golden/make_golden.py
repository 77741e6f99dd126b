"""Generate golden fixtures by running the UNMODIFIED reference ``parafrac``.

Run here (the reference is importable read-only from /root/reference); the
fixtures travel with the repo, the reference does not:

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Contents of ``reference_goldens.npz`` (all float64 unless noted):

* the reference test-suite known answers re-derived by running the reference:
  ``u1_paper42_nt4_n8`` (first coarse step, test_stepping.py:29-33,64-68),
  ``coarse_norm_nt64_n8`` (test_stepping.py:34,107-109),
  ``fine_endpoint_n0_m4_n8`` (test_stepping.py:35-39,134-139),
  ``fine_norm_nt64_m8_n16`` (test_stepping.py:40,192-194),
  ``l2_ones_op16`` (test_spectral.py:117-121);
* paper42 on degree 8 / 16: run_coarse, fine sweep, chain_fine,
  run_fine_sequential and a full parareal run (iterates, diffs, caches);
* BASELINE configs 1 and 2 in the reference's own Chebyshev form (degree
  M+1, same P, m, alpha, T, D, f, u0): parareal iterates, diff sequence and
  iteration count to tol 1e-12.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = os.environ.get("PARAFRAC_REFERENCE", "/root/reference/pkg/src")


def _sine_series(amps):
    amps = np.asarray(amps, dtype=float)
    k = np.arange(1, amps.size + 1)

    def initial(x):
        x = np.asarray(x, dtype=float)
        return np.sin(np.pi * np.multiply.outer(x, k)) @ amps

    return initial


def cfg_problem_cheb(pf, i):
    """Configs 1-2 as reference ProblemSpecs (numpy callbacks)."""
    def d12(x, t, u):
        return 1.0 + u**2 / (1.0 + u**2)

    def f12(x, t, u):
        return np.sin(np.pi * x) * np.cos(u)

    if i == 1:
        M = 32
        amps = np.zeros(M)
        amps[0], amps[2] = 1.0, 0.5
        return pf.ProblemSpec(0.0, 1.0, 1.0, 0.5, d12, f12, _sine_series(amps), name="cfg1")
    M = 64
    k = np.arange(1, M + 1, dtype=float)
    amps = np.random.default_rng(1).standard_normal(M) * k ** -3.0
    return pf.ProblemSpec(0.0, 1.0, 1.0, 1.0, d12, f12, _sine_series(amps), name="cfg2")


def main():
    sys.path.insert(0, REF)
    import parafrac as pf
    from parafrac.parareal import _solve
    from parafrac.stepping import fine_sweep_intervals

    out = {}
    p42 = pf.get_problem("paper42")
    op8 = pf.build_operator(8, 0.0, 1.0)
    op16 = pf.build_operator(16, 0.0, 1.0)
    g = pf.TimeGrids(1.0, 4, 1)
    u0 = pf.initial_state(p42, op8)
    out["u1_paper42_nt4_n8"] = pf.coarse_step(u0[None, :], op8, g, p42)
    out["coarse_norm_nt64_n8"] = np.array(pf.l2_norm(op8, pf.run_coarse(p42, op8, pf.TimeGrids(1.0, 64, 1))[-1]))
    out["fine_endpoint_n0_m4_n8"] = pf.fine_propagate(u0, u0[None, :], op8, pf.TimeGrids(1.0, 4, 4), p42)[0]
    seq, _ = pf.run_fine_sequential(p42, op16, pf.TimeGrids(1.0, 64, 8))
    out["fine_norm_nt64_m8_n16"] = np.array(pf.l2_norm(op16, seq[-1]))
    out["l2_ones_op16"] = np.array(pf.l2_norm(op16, np.ones(15)))

    for deg, nt, m in ((8, 8, 4), (16, 16, 4)):
        op = pf.build_operator(deg, 0.0, 1.0)
        gr = pf.TimeGrids(1.0, nt, m)
        tag = f"p42_d{deg}_nt{nt}_m{m}"
        traj = pf.run_coarse(p42, op, gr)
        out[f"{tag}_run_coarse"] = traj
        out[f"{tag}_fine_sweep"] = fine_sweep_intervals(traj, 0, nt, op, gr, p42)
        out[f"{tag}_chain_fine"] = pf.chain_fine(p42, op, gr)
        out[f"{tag}_fine_sequential"] = pf.run_fine_sequential(p42, op, gr)[0]
        it, rep = _solve(p42, op, gr, tol=1e-12, k_max=nt + 1, threads=1, reference=None)
        out[f"{tag}_states"] = it.states
        out[f"{tag}_coarse_new"] = it.coarse_new
        out[f"{tag}_coarse_old"] = it.coarse_old
        out[f"{tag}_fine_endpoints"] = it.fine_endpoints
        out[f"{tag}_diffs"] = np.array(rep.diffs)
        out[f"{tag}_iterations"] = np.array(rep.iterations)

    for i, (deg, nt, m, alpha) in ((1, (33, 8, 64, 0.5)), (2, (65, 16, 256, 1.0))):
        prob = cfg_problem_cheb(pf, i)
        op = pf.build_operator(deg, 0.0, 1.0)
        gr = pf.TimeGrids(1.0, nt, m)
        it, rep = _solve(prob, op, gr, tol=1e-12, k_max=nt + 1, threads=1, reference=None)
        out[f"cheb_cfg{i}_states"] = it.states
        out[f"cheb_cfg{i}_diffs"] = np.array(rep.diffs)
        out[f"cheb_cfg{i}_iterations"] = np.array(rep.iterations)
        out[f"cheb_cfg{i}_chain_fine"] = pf.chain_fine(prob, op, gr)

    path = os.path.join(HERE, "reference_goldens.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {len(out)} arrays, {os.path.getsize(path)} bytes")
    for k in ("cheb_cfg1_iterations", "cheb_cfg2_iterations"):
        print(k, int(out[k]))


if __name__ == "__main__":
    main()
