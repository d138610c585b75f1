"""Shared fixtures: golden data produced by the reference (tests/golden/make_golden.py)."""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")

# BASELINE.json tolerances, written where they are used:
#   elementwise L parity, scale max(|L_ref|, 1) (pkg/tests/test_acceptance.py:49)
L_TOL = 1e-10
#   backward error ||A - L L^T||_F / ||A||_F <= 10 * n * eps
EPS = float(np.finfo(np.float64).eps)
#   solve: ||x - x_ref|| / ||x_ref|| (pkg/tests/test_core.py:214-220)
X_TOL = 1e-10


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running full-size check")


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="session")
def golden_meta():
    with open(os.path.join(GOLDEN, "fingerprints.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def small():
    with np.load(os.path.join(GOLDEN, "small_cases.npz")) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def large():
    with np.load(os.path.join(GOLDEN, "sampled_large.npz")) as z:
        return {k: z[k] for k in z.files}


def scaled_diff(got: np.ndarray, want: np.ndarray) -> float:
    """max |got - want| / max(|want|, 1) -- the reference's parity scale."""
    scale = np.maximum(np.abs(want), 1.0)
    return float(np.max(np.abs(got - want) / scale)) if want.size else 0.0


def band_panel(n, k, ld, data):
    p = data.reshape(n, ld).T[: k + 1].copy()
    for d in range(1, k + 1):
        p[d, n - d:] = 0.0
    return p


def band_matvec(n, k, ld, data, x):
    """y = A x for a symmetric band matrix in lower band storage (vectorised)."""
    p = data.reshape(n, ld).T
    y = p[0, :n] * x
    for d in range(1, k + 1):
        y[d:] += p[d, : n - d] * x[: n - d]
        y[: n - d] += p[d, : n - d] * x[d:]
    return y


def band_matvec_batched(n, k, ld, data, x):
    """Row-wise batched band matvec: data (B, ld*n), x (B, n)."""
    p = data.reshape(data.shape[0], n, ld)
    y = p[:, :, 0] * x
    for d in range(1, k + 1):
        y[:, d:] += p[:, : n - d, d] * x[:, : n - d]
        y[:, : n - d] += p[:, : n - d, d] * x[:, d:]
    return y
