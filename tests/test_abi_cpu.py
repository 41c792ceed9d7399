"""CPU-only checks of the boundary: the C-ABI library loads and exports every
function declared in include/pdsdp_b200.h; argument validation that needs no
GPU; host-side control logic mirrors the reference (lowrank.py:64-83)."""

import os
import re
import ctypes as ct
from collections import deque

import numpy as np
import pytest

from conftest import ROOT
from paper_1810_05231_b200 import device
from paper_1810_05231_b200.config import (
    RankController, SolverConfig, rank_certificate_satisfied, stall_detected, update_rank,
)
from paper_1810_05231_b200.layout import approx_error_bound, packed_index, smat, svec, SymMatrix


def header_functions():
    txt = open(os.path.join(ROOT, "include", "pdsdp_b200.h")).read()
    return sorted(set(re.findall(r"\b(pdsdp_[a-z_A-Z0-9]+)\s*\(", txt)))


def test_library_exports_every_header_symbol():
    lib = ct.CDLL(device.LIB_PATH)
    names = header_functions()
    assert len(names) >= 15
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(device.EXPORTED)


def test_library_reports_version_and_errors_without_gpu():
    lib = device.load_library()
    assert lib.pdsdp_version() == 1
    assert lib.pdsdp_strerror(-1) == b"invalid argument"
    # invalid arguments are rejected before any device work
    assert lib.pdsdp_aproj_psd(0, None, 1, None, None) == device.EINVAL
    assert lib.pdsdp_batch_create(0, None, None) == device.EINVAL


def test_stall_rule_matches_reference_examples():
    # SPEC lowrank examples; reference lowrank.py:64-69
    assert not stall_detected(deque([5, 4, 3, 2]), 3)
    assert stall_detected(deque([1, 1, 1, 1]), 3)
    assert not stall_detected(deque([1, 1]), 3)


def test_update_rank_and_certificate():
    c = RankController(r=3, ell=4, history=deque([1.0, 2.0]))
    assert update_rank(c, 5) == 5 and len(c.history) == 0
    assert update_rank(c, 5) == 5
    assert rank_certificate_satisfied(10, 10, 2.0, 0.0)
    assert rank_certificate_satisfied(10, 4, -0.5, 0.0)
    assert not rank_certificate_satisfied(100, 4, 0.01, 0.5)
    assert approx_error_bound(10, 4, 0.5) == pytest.approx(3.0)
    with pytest.raises(ValueError):
        approx_error_bound(5, 0, 1.0)


def test_config_validation_messages():
    for kw, msg in [({"eps_tol": 0}, "eps_tol"), ({"alpha_safety": 1.0}, "alpha_safety"),
                    ({"window_ell": 0}, "window_ell"), ({"initial_rank": 0}, "initial_rank"),
                    ({"alpha_override": -1.0}, "alpha_override"), ({"progress_every": 0}, "progress_every")]:
        with pytest.raises(ValueError, match=msg):
            SolverConfig(**kw).validate()


def test_packed_layout_round_trip(rng):
    for n in (1, 2, 7):
        R = rng.standard_normal((n, n))
        S = R + R.T
        v = svec(S)
        assert np.allclose(smat(v), S)
        if n > 1:
            assert v[packed_index(n, 0, 1)] == pytest.approx(np.sqrt(2) * S[0, 1])
        A = SymMatrix.from_dense(S)
        assert A.inner(A) == pytest.approx(np.trace(S @ S))
    with pytest.raises(ValueError, match="not symmetric"):
        svec(np.array([[1.0, 2.0], [0.0, 1.0]]))
