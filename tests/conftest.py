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
