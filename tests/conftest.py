"""Shared fixtures.  ``-m "not gpu"`` runs here (no GPU); ``-m gpu`` runs on a B200."""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN_PATH = os.path.join(ROOT, "tests", "golden", "reference_goldens.npz")
REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the sm_100a C-ABI library)")


@pytest.fixture(scope="session")
def golden():
    with np.load(GOLDEN_PATH) as z:
        return {k: z[k] for k in z.files}


def reference_available():
    return os.path.isdir(REFERENCE_SRC)


def rel_err(a, b):
    a = np.asarray(a, dtype=float)
    b = np.asarray(b, dtype=float)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def sine_u(coeffs, x):
    """Evaluate sum_k c_k sqrt(2) sin(k pi x) (sine-Galerkin state -> grid)."""
    k = np.arange(1, coeffs.shape[-1] + 1)
    return (np.sqrt(2.0) * np.sin(np.pi * np.multiply.outer(np.asarray(x), k))) @ np.asarray(coeffs).T
