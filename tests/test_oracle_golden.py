"""Pin the CPU oracle against outputs of the reference itself (CPU only).

Fixtures come from tests/golden/make_golden.py, which ran the unmodified
reference package; plus the known-answer cases of the reference's own tests
(``pkg/tests/test_symmat.py:197-209``, ``test_pdhg.py:35-75``).
"""

import numpy as np
import pytest

from conftest import load_golden, problem_from_golden
from oracle import lrpdhg_oracle as orc
from paper_1810_05231_b200 import workloads
from paper_1810_05231_b200.config import SolverConfig


def test_known_answer_aproj_diag():
    # reference test_symmat.py:197-201: aproj(diag(5,3,-1), 1) -> diag(5,0,0), lambda = 3
    S = orc.pack(np.diag([5.0, 3.0, -1.0]))
    P, lam = orc.aproj_psd(S, 3, 1)
    np.testing.assert_allclose(orc.unpack(P, 3), np.diag([5.0, 0, 0]), atol=1e-12)
    assert lam == pytest.approx(3.0)


def test_known_answer_box_resolvent():
    # reference test_pdhg.py:62-69
    out = orc.box_resolvent(np.array([4.0]), 1.0, np.array([1.0]), np.zeros(0))
    np.testing.assert_allclose(out, [3.0])
    out = orc.box_resolvent(np.array([4.0]), 2.0, np.array([1.0]), np.zeros(0))
    np.testing.assert_allclose(out, [2.0])


@pytest.mark.parametrize("ci", range(5))
def test_ops_match_reference(ci):
    d = load_golden("ops_small.npz")
    pre = f"c{ci}_"
    prob = problem_from_golden(d, pre)
    n = prob.n
    M = orc.stacked_csr(prob)
    np.testing.assert_allclose(M @ d[pre + "X"], d[pre + "MX"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(M.T @ d[pre + "y"], d[pre + "MTy"], rtol=0, atol=1e-12)
    assert orc.op_norm(M, 0) == pytest.approx(float(d[pre + "opnorm"]), rel=1e-12)
    for r in (1, 3, n // 2, n):
        P, lam = orc.aproj_psd(d[pre + "S"], n, r)
        np.testing.assert_allclose(P, d[pre + f"aproj{r}"], atol=1e-9)
        assert lam == pytest.approx(float(d[pre + f"aproj{r}_lam"]), abs=1e-9)
    w, _, _ = orc.top_eigen(d[pre + "S"], n, min(5, n))
    np.testing.assert_allclose(w, d[pre + "teig_vals"], atol=1e-9)
    alpha = 0.37
    yn = orc.dual_update(M, d[pre + "y"], d[pre + "Xn"], d[pre + "X"], alpha, prob.b, prob.h)
    np.testing.assert_allclose(yn, d[pre + "dual"], atol=1e-12)
    res = orc.fixed_point_residuals(M, d[pre + "Xn"], d[pre + "X"], yn, d[pre + "y"], alpha)
    np.testing.assert_allclose(res, d[pre + "resid"], rtol=1e-12)


@pytest.mark.parametrize("ci", range(5))
def test_lr_small_solves_match_reference(ci):
    d = load_golden("lr_small.npz")
    pre = f"c{ci}_"
    prob = problem_from_golden(d, pre)
    cfg = SolverConfig(eps_tol=1e-4, max_iter=400, initial_rank=int(d[pre + "r0"]),
                       window_ell=50, time_limit_s=1e9)
    res = orc.solve_lr(prob, cfg)
    assert res.status == str(d[pre + "status"])
    assert res.iterations == int(d[pre + "iters"])
    assert [tuple(x) for x in res.rank_path] == [tuple(x) for x in d[pre + "rank_path"].tolist()]
    scale = np.linalg.norm(d[pre + "X"])
    assert np.linalg.norm(res.X - d[pre + "X"]) <= 1e-8 * scale
    assert res.primal_objective == pytest.approx(float(d[pre + "pobj"]), rel=1e-8)


def test_config1_matches_reference():
    d = load_golden("cfg1.npz")
    prob, cfg = workloads.config(0)
    np.testing.assert_array_equal(prob.C.data, d["C"])
    res = orc.solve_lr(prob, cfg, record_at=(1, 10, 100))
    assert res.status == "optimal" == str(d["status"])
    assert res.iterations == int(d["iters"]) == 1718
    assert res.rank_path == [tuple(x) for x in d["rank_path"].tolist()]
    for K in (1, 10, 100):
        X, y, lam, r = res.snapshots[K]
        assert np.linalg.norm(X - d[f"X{K}"]) <= 1e-10 * np.linalg.norm(d[f"X{K}"])
        assert np.linalg.norm(y - d[f"y{K}"]) <= 1e-10 * np.linalg.norm(d[f"y{K}"])
        assert lam == pytest.approx(float(d[f"lam{K}"]), rel=1e-8, abs=1e-10)
    assert np.linalg.norm(res.X - d["X_final"]) <= 1e-8 * np.linalg.norm(d["X_final"])
    assert res.primal_objective == pytest.approx(float(d["pobj"]), rel=1e-10)
    hist = np.array(res.history)
    np.testing.assert_allclose(hist[:, 2], d["history"][:, 3], rtol=1e-7)


@pytest.mark.parametrize("ci", range(4))
def test_exact_pd_oracle_matches_reference(ci):
    d = load_golden("pd_small.npz")
    pre = f"c{ci}_"
    prob = problem_from_golden(d, pre)
    for K in (1, 10):
        r = orc.solve_pd(prob, SolverConfig(eps_tol=1e-4, max_iter=K, time_limit_s=1e9))
        assert np.linalg.norm(r.X - d[pre + f"X{K}"]) <= 1e-10 * max(1.0, np.linalg.norm(d[pre + f"X{K}"]))
        assert np.linalg.norm(r.y - d[pre + f"y{K}"]) <= 1e-10 * max(1.0, np.linalg.norm(d[pre + f"y{K}"]))
    if prob.n <= 30:    # the full runs of the small cases (the n = 48 case runs 3000 iterations)
        r = orc.solve_pd(prob, SolverConfig(eps_tol=1e-4, max_iter=3000, time_limit_s=1e9))
        assert r.status == str(d[pre + "status"]) and r.iterations == int(d[pre + "iters"])
        assert r.primal_objective == pytest.approx(float(d[pre + "pobj"]), rel=1e-9, abs=1e-12)


def test_mimo_oracle_matches_reference():
    d = load_golden("mimo.npz")
    pre = "c0_"
    prob = problem_from_golden(d, pre)
    K = int(d[pre + "K"])
    r = orc.solve_lr(prob, SolverConfig(eps_tol=1e-4, max_iter=K, initial_rank=1, window_ell=50,
                                        time_limit_s=1e9))
    assert r.status == str(d[pre + "status"]) and r.iterations == int(d[pre + "iters"])
    assert [tuple(x) for x in r.rank_path] == [tuple(x) for x in d[pre + "rank_path"].tolist()]
    assert np.linalg.norm(r.X - d[pre + "X"]) <= 1e-8 * np.linalg.norm(d[pre + "X"])


def test_check_solution_oracle_matches_reference():
    d = load_golden("check.npz")
    keys = sorted({"_".join(k.split("_")[:2]) + "_" for k in d.files if k.startswith("k")})
    for q in keys:
        prob = problem_from_golden(d, q)
        got = orc.check_solution(prob, d[q + "X"], d[q + "yv"])
        np.testing.assert_allclose(got, d[q + "report"], rtol=1e-10, atol=1e-12)
