"""The drop-in accepts reference-typed inputs (VERDICT r01 'missing' #3).

CPU part: real ``pdsdp.SdpProblem`` objects (imported from /root/reference in
this test only -- the package never imports the reference; skipped where the
reference tree is absent, e.g. on the GPU box) convert by duck typing into the
same C-ABI problem descriptor, and this package's ``SolveStatus`` is accepted
by the reference's own status table (``cli.py:178-186``)."""

import importlib
import os
import sys

import numpy as np
import pytest

import paper_1810_05231_b200 as pk
from paper_1810_05231_b200 import workloads
from paper_1810_05231_b200.model import as_problem

REF_SRC = "/root/reference/pkg/src"


@pytest.fixture(scope="module")
def pdsdp():
    if not os.path.isdir(REF_SRC):
        pytest.skip("reference tree not present")
    sys.path.insert(0, REF_SRC)
    try:
        return importlib.import_module("pdsdp")
    finally:
        sys.path.remove(REF_SRC)


def _ref_problem(pdsdp, prob):
    return pdsdp.SdpProblem(
        n=prob.n, C=pdsdp.SymMatrix(prob.n, prob.C.data.copy()),
        A=[pdsdp.SparseRow(r.indices, r.values) for r in prob.A], b=prob.b.copy(),
        G=[pdsdp.SparseRow(r.indices, r.values) for r in prob.G], h=prob.h.copy(),
        name=prob.name, objective_sign=-1.0)


def test_reference_problem_converts_to_same_descriptor(pdsdp):
    rng = np.random.default_rng(3)
    ours = workloads.maxcut_problem(40, 0.2, 7, signed=True)
    G = [pk.SparseRow.from_matrix_entries(40, [(1, 5, 0.5), (2, 2, 1.0)])]
    ours = pk.SdpProblem(n=40, C=ours.C, A=ours.A, b=ours.b, G=G, h=rng.standard_normal(1))
    ref = _ref_problem(pdsdp, ours)
    conv = as_problem(ref)
    assert isinstance(conv, pk.SdpProblem) and conv is as_problem(ref)      # cached off-object
    assert not hasattr(ref, "_device_cache")
    assert (conv.n, conv.m, conv.p, conv.objective_sign) == (40, 40, 1, -1.0)
    for a, b in zip(conv.stacked_arrays(), ours.stacked_arrays()):
        assert np.array_equal(a, b)
    # the reference's own CSR (problem.py:119-137) holds the same operator
    M = ref.stacked()
    ip, ix, vv = conv.stacked_arrays()
    assert np.array_equal(M.indptr, ip) and np.array_equal(M.indices, ix) and np.array_equal(M.data, vv)
    assert np.array_equal(conv.C.data, ref.C.data) and np.array_equal(conv.b, ref.b)
    assert np.array_equal(conv.h, ref.h)


def test_conversion_cache_is_released_with_the_object(pdsdp):
    from paper_1810_05231_b200 import model
    ref = _ref_problem(pdsdp, workloads.maxcut_problem(10, 0.5, 1, signed=False))
    as_problem(ref)
    key = id(ref)
    assert key in model._converted
    del ref
    import gc
    gc.collect()
    assert key not in model._converted


def test_status_is_accepted_by_reference_tables(pdsdp):
    cli = importlib.import_module("pdsdp.cli")
    ref_status = importlib.import_module("pdsdp.pdhg").SolveStatus
    for name in ("OPTIMAL", "MAX_ITERATIONS", "TIME_LIMIT", "DIVERGED"):
        mine, theirs = getattr(pk.SolveStatus, name), getattr(ref_status, name)
        assert cli._status_exit_code(mine) == cli._status_exit_code(theirs)
        assert mine == theirs and theirs == mine and hash(mine) == hash(theirs)
        assert mine.value == theirs.value
    assert pk.SolveStatus.OPTIMAL != ref_status.DIVERGED
    assert pk.SolveStatus.OPTIMAL != "optimal"
    assert len({pk.SolveStatus.OPTIMAL, pk.SolveStatus.DIVERGED}) == 2


def test_reference_config_is_accepted_by_validation(pdsdp):
    cfg = pdsdp.SolverConfig(eps_tol=1e-4, initial_rank=3)
    cfg.validate()
    ours = pk.SolverConfig(eps_tol=1e-4, initial_rank=3)
    assert {k: getattr(cfg, k) for k in ours.__dict__} == ours.__dict__


def test_non_problem_is_rejected():
    with pytest.raises(TypeError, match="SdpProblem-like"):
        as_problem(object())
