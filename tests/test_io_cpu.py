"""problem / solution documents at the boundary, against
the reference's own io.py outputs (tests/golden/io.npz, make_golden.py)."""

import json

import numpy as np
import pytest

from conftest import load_golden, problem_from_golden
from paper_1810_05231_b200 import io as bio
from paper_1810_05231_b200.config import Checkpoint, SolutionReport, SolveResult, SolveStatus
from paper_1810_05231_b200.layout import SymMatrix


def _same_problem(p, d, pre):
    ref = problem_from_golden(d, pre)
    assert p.n == ref.n and p.m == ref.m and p.p == ref.p
    np.testing.assert_array_equal(p.C.data, ref.C.data)
    np.testing.assert_array_equal(p.b, ref.b)
    np.testing.assert_array_equal(p.h, ref.h)
    for a, b in zip(list(p.A) + list(p.G), list(ref.A) + list(ref.G)):
        np.testing.assert_array_equal(a.indices, b.indices)
        np.testing.assert_array_equal(a.values, b.values)


@pytest.mark.parametrize("name", ["cfg1", "multi"])
def test_sdpa_parse_and_rewrite_match_reference(name):
    d = load_golden("io.npz")
    pre = f"sdpa_{name}_"
    p = bio.parse_sdpa(str(d[pre + "text"]))
    _same_problem(p, d, pre)
    assert p.objective_sign == float(d[pre + "sign"]) == -1.0
    assert bio.write_sdpa(p) == str(d[pre + "rewrite"])


def test_sdpa_errors_match_reference():
    d = load_golden("io.npz")
    for text, msg in zip(d["sdpa_bad_text"], d["sdpa_bad_msg"]):
        with pytest.raises(bio.ParseError) as exc:
            bio.parse_sdpa(str(text))
        assert str(exc.value) == str(msg)


def test_extended_roundtrip_matches_reference():
    d = load_golden("io.npz")
    text = str(d["ext_text"])
    p = bio.parse_extended(text)
    _same_problem(p, d, "ext_")
    assert p.name == "lr_small_c1"
    assert json.loads(bio.write_extended(p)) == json.loads(text)


def test_solution_document_roundtrip():
    d = load_golden("io.npz")
    text = str(d["sol_text"])
    doc = bio.read_solution(text)
    res = SolveResult(status=SolveStatus(doc["status"]), X=doc["X"], y=doc["y"],
                      primal_objective=doc["primal_objective"], dual_objective=doc["dual_objective"],
                      final_residuals=(doc["residuals"]["primal"], doc["residuals"]["dual"],
                                       doc["residuals"]["combined"]),
                      iterations=doc["iterations"], rank_path=[tuple(x) for x in doc["rank_path"]],
                      checkpoints=[Checkpoint(c["rank"], doc["X"], doc["y"], c["objective"]) for c in doc["checkpoints"]],
                      wall_time_s=doc["wall_time_s"], residual_scale=doc["residuals"]["scale"],
                      objective_sign=doc["objective_sign"])
    rep = SolutionReport(doc["primal_objective"], doc["dual_objective"], doc["equality_violation"],
                         doc["inequality_violation"], doc["min_eigenvalue"], doc["duality_gap"])
    assert json.loads(bio.write_solution(res, rep)) == json.loads(text)
    with pytest.raises(bio.ParseError):
        bio.read_solution('{"format": "other"}')


def test_load_problem_detects_format(tmp_path):
    d = load_golden("io.npz")
    f = tmp_path / "x.dat-s"
    f.write_text(str(d["sdpa_multi_text"]))
    p = bio.load_problem(f)
    assert p.name == "x.dat-s" and p.n == 5
    with pytest.raises(ValueError, match="cannot infer"):
        bio.load_problem(tmp_path / "x.txt")
