"""Inter-CTA protocol under perturbed timing (``-m gpu``).

The fine sweep's slice and helper CTAs exchange far-history blocks through
release/acquire flags (pf_kernels.cuh ``cta_publish`` / ``ld_acquire``).
compute-sanitizer is closed on this pool (profiles/r02_compute_sanitizer_closed.txt),
so the protocol is checked by a stress build instead: ``-DPF_JITTER`` makes
every slice CTA delay its progress publish and every helper CTA its block by a
pseudo-random 0..8 us.  Under any interleaving the sweep must be bitwise the
inline far history (PF_NO_HELPERS=1, no inter-CTA protocol at all), and the
sequential solver with its far history split over several helper CTAs
(per-batch tickets, last arrival combines) bitwise the regular build."""

import os
import subprocess
import sys
import tempfile

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
JITTER = os.path.join(ROOT, "paper_2510_11023_b200", "libparafrac_b200_jitter.so")

CODE = """
import sys, numpy as np
sys.path.insert(0, {root!r})
import paper_2510_11023_b200 as p
from paper_2510_11023_b200 import _lib
pr = p.config_problem(3); op = p.build_sine_operator(512)
g = p.TimeGrids(2.0, 16, 96)
t = p.run_coarse(pr, op, g)
out = p.fine_sweep_intervals(t, 0, 16, op, g, pr)
ctx = _lib.context_for(pr, op, g)
seq, _ = p.run_fine_sequential(pr, op, p.TimeGrids(2.0, 4, 128))
g2 = p.TimeGrids(2.0, 4, 1024)  # 4096 substeps: the far history split over 4 helper CTAs
seq2, _ = p.run_fine_sequential(pr, op, g2)
np.savez(sys.argv[1], sweep=out, seq=seq, seq2=seq2, helpers=ctx.stats()["helper_launches"],
         helpers2=_lib.context_for(pr, op, g2).stats()["helper_launches"], lib=_lib.LIB_PATH)
"""


def _run(env_extra):
    with tempfile.TemporaryDirectory() as d:
        f = os.path.join(d, "o.npz")
        subprocess.run([sys.executable, "-c", CODE.format(root=ROOT), f], check=True,
                       env=dict(os.environ, **env_extra))
        z = np.load(f)
        return {k: z[k] for k in z.files}


def test_handshake_bitwise_under_jitter():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a B200")
    if not os.path.exists(JITTER):
        pytest.fail("the -DPF_JITTER build is missing: run __graft_entry__.build()")
    jit = _run({"PARAFRAC_B200_LIB": JITTER})
    assert str(jit["lib"]).endswith("libparafrac_b200_jitter.so")
    assert int(jit["helpers"]) >= 1  # the cooperative slice + helper launch ran
    inline = _run({"PF_NO_HELPERS": "1"})
    assert int(inline["helpers"]) == 0
    np.testing.assert_array_equal(jit["sweep"], inline["sweep"])
    plain = _run({})
    np.testing.assert_array_equal(plain["sweep"], inline["sweep"])
    np.testing.assert_array_equal(jit["seq"], plain["seq"])
    # the split tensor-core helpers of the sequential solver: deterministic under
    # jitter, and the same sums as the inline far history up to rounding order
    assert int(jit["helpers2"]) >= 1 and int(inline["helpers2"]) == 0
    np.testing.assert_array_equal(jit["seq2"], plain["seq2"])
    assert np.linalg.norm(plain["seq2"] - inline["seq2"]) <= 1e-12 * np.linalg.norm(inline["seq2"])


@pytest.mark.parametrize("far_tc", ["1", "2"])
def test_tensor_core_far_history_helper_bitwise_inline(far_tc):
    """PF_FAR_TC=1 (DMMA, direct loads) / 2 (DMMA fed by TMA bulk copies, the old
    rows accumulated for four tiles per pass: the default at M = 512): the
    helper CTA's far history under jitter == the slice CTA's inline DMMA path,
    bitwise, and the DFMA engine (PF_FAR_TC=0) to rounding."""
    import torch

    if not torch.cuda.is_available():
        pytest.fail("gpu tests need a B200")
    helper = _run({"PARAFRAC_B200_LIB": JITTER, "PF_FAR_TC": far_tc})
    inline = _run({"PF_NO_HELPERS": "1", "PF_FAR_TC": "1"})
    assert int(helper["helpers"]) >= 1 and int(inline["helpers"]) == 0
    np.testing.assert_array_equal(helper["sweep"], inline["sweep"])
    dfma = _run({"PF_FAR_TC": "0"})
    assert np.linalg.norm(helper["sweep"] - dfma["sweep"]) <= 1e-13 * np.linalg.norm(dfma["sweep"])
    if far_tc == "2":
        # engine 2 is the default at M = 512 (grouped passes over the old rows, TC_G tiles per pass)
        assert np.array_equal(_run({})["sweep"], helper["sweep"])
        # the DFMA register-tile helper (PF_FAR_TC=0) under jitter == its inline path, bitwise
        dfma_jit = _run({"PARAFRAC_B200_LIB": JITTER, "PF_FAR_TC": "0"})
        dfma_inline = _run({"PF_NO_HELPERS": "1", "PF_FAR_TC": "0"})
        assert int(dfma_jit["helpers"]) >= 1 and int(dfma_inline["helpers"]) == 0
        np.testing.assert_array_equal(dfma_jit["sweep"], dfma_inline["sweep"])
        np.testing.assert_array_equal(dfma["sweep"], dfma_inline["sweep"])
