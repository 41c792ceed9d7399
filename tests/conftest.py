"""Shared fixtures: golden-fixture loading and problem reconstruction."""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")

from paper_1810_05231_b200.layout import SymMatrix  # noqa: E402
from paper_1810_05231_b200.model import SdpProblem, SparseRow  # noqa: E402


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through the CUDA C-ABI)")
    config.addinivalue_line("markers", "slow: long-running")


def load_golden(name):
    path = os.path.join(GOLDEN, name)
    if not os.path.exists(path):
        pytest.skip(f"golden fixture {name} not generated")
    return np.load(path, allow_pickle=False)


def problem_from_golden(d, prefix="") -> SdpProblem:
    n = int(d[prefix + "n"])
    indptr = d[prefix + "indptr"]
    idx, val = d[prefix + "idx"], d[prefix + "val"]
    b, h = d[prefix + "b"], d[prefix + "h"]
    rows = [SparseRow(idx[indptr[i]:indptr[i + 1]], val[indptr[i]:indptr[i + 1]])
            for i in range(len(indptr) - 1)]
    m = b.size
    return SdpProblem(n=n, C=SymMatrix(n, d[prefix + "C"]), A=rows[:m], b=b,
                      G=rows[m:], h=h)


@pytest.fixture
def rng():
    return np.random.default_rng(12345)


def dense_case_matrix(n, seed):
    """Seeded symmetric test matrix of the dense-eigensolver fixtures
    (tests/golden/make_golden.py make_dense builds the same one): random
    symmetric plus a few planted large eigenvalues, so kept / clipped /
    certificate pairs are all present."""
    rng = np.random.default_rng(seed)
    R = rng.standard_normal((n, n))
    S = 0.5 * (R + R.T) / np.sqrt(n)
    U = rng.standard_normal((n, 5))
    return S + (U * np.array([4.0, 3.0, 2.5, -3.5, 2.0])) @ U.T / n
