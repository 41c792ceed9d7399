"""GPU parity: the sm_100a path (through the C ABI) against the reference's
own outputs (golden fixtures from tests/golden/make_golden.py) and the CPU
oracle on the same seeded inputs.

Tolerances are the north star's (BASELINE.json): iterates within 1e-8
relative Frobenius at a fixed iteration count, objectives within 1e-5
relative, the same 1e-4 stopping rule met at the same iteration.  Integer /
index outputs (iteration counts, rank paths, statuses) must match exactly.
"""

import numpy as np
import pytest

from conftest import load_golden, problem_from_golden
from oracle import lrpdhg_oracle as orc
import paper_1810_05231_b200 as pk
from paper_1810_05231_b200 import workloads
from paper_1810_05231_b200.config import SolverConfig

pytestmark = pytest.mark.gpu

ITER_TOL = 1e-8      # relative Frobenius, fixed K
OBJ_TOL = 1e-5       # relative objective


def rel(a, b, floor=1e-12):
    """Relative error; references that are zero up to rounding (e.g. X+ = 0
    when S is negative semidefinite) are compared absolutely against `floor`."""
    nb = np.linalg.norm(b)
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(nb, floor)


def with_iters(cfg, K, **kw):
    return SolverConfig(**{**cfg.__dict__, "max_iter": K, **kw})


# ---------------------------------------------------------------- op level

@pytest.mark.parametrize("ci", range(5))
def test_linear_maps_and_opnorm(ci):
    d = load_golden("ops_small.npz")
    pre = f"c{ci}_"
    prob = problem_from_golden(d, pre)
    n = prob.n
    mx = pk.apply_M(prob, pk.SymMatrix(n, d[pre + "X"]))
    np.testing.assert_allclose(mx, d[pre + "MX"], rtol=0, atol=1e-12)
    mty = pk.apply_M_adjoint(prob, d[pre + "y"]).data
    np.testing.assert_allclose(mty, d[pre + "MTy"], rtol=0, atol=1e-12)
    assert pk.estimate_operator_norm(prob, 0) == pytest.approx(float(d[pre + "opnorm"]), rel=1e-12)


@pytest.mark.parametrize("ci", range(5))
def test_aproj_psd_matches_reference(ci):
    d = load_golden("ops_small.npz")
    pre = f"c{ci}_"
    n = int(d[pre + "n"])
    S = pk.SymMatrix(n, d[pre + "S"])
    for r in (1, 3, n // 2, n):
        P, lam = pk.aproj_psd(S, r)
        ref = d[pre + f"aproj{r}"]
        assert rel(P.data, ref) <= ITER_TOL
        assert lam == pytest.approx(float(d[pre + f"aproj{r}_lam"]), rel=1e-9, abs=1e-11)


def test_aproj_known_answer_and_errors():
    # reference test_symmat.py:197-201 (pins lambda_{r+1})
    P, lam = pk.aproj_psd(pk.SymMatrix.from_dense(np.diag([5.0, 3.0, -1.0])), 1)
    np.testing.assert_allclose(P.to_dense(), np.diag([5.0, 0.0, 0.0]), atol=1e-12)
    assert lam == pytest.approx(3.0)
    with pytest.raises(ValueError, match="outside"):
        pk.aproj_psd(pk.SymMatrix.from_dense(np.eye(3)), 0)
    with pytest.raises(ValueError, match="outside"):
        pk.aproj_psd(pk.SymMatrix.from_dense(np.eye(3)), 4)


def test_aproj_random_vs_oracle(rng):
    for n, r in ((33, 4), (80, 7), (150, 12), (300, 20)):
        R = rng.standard_normal((n, n))
        S = orc.pack(0.5 * (R + R.T))
        P, lam = pk.aproj_psd(pk.SymMatrix(n, S), r)
        Pr, lr = orc.aproj_psd(S, n, r)
        assert rel(P.data, Pr) <= ITER_TOL
        assert lam == pytest.approx(lr, rel=1e-8)


def test_aproj_clustered_spectrum_vs_oracle(rng):
    """Repeated and nearly repeated kept eigenvalues (the Jacobi pairs with
    ~zero gap must take the rotation path, not the second-order finish) and a
    negative tail; X+ is basis-independent within each cluster."""
    for n, r in ((64, 6), (200, 10), (400, 21)):
        Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
        lam = -rng.random(n)
        top = np.concatenate([[9.0, 9.0, 9.0 * (1 + 1e-9), 4.0, 4.0 + 1e-7, 2.0], 1.0 + rng.random(r)])[:r]
        lam[:r] = top
        D = (Q * lam) @ Q.T
        S = orc.pack(0.5 * (D + D.T))
        P, lm = pk.aproj_psd(pk.SymMatrix(n, S), r)
        Pr, lr = orc.aproj_psd(S, n, r)
        assert rel(P.data, Pr) <= ITER_TOL
        assert lm == pytest.approx(lr, rel=1e-8, abs=1e-10)


def test_aproj_triple_clusters_vs_oracle(rng):
    """Three or more nearly equal kept eigenvalues (relative gaps 1e-10 ..
    1e-12): the Jacobi second-order finish U = I + K loses orthogonality by
    K^T K there, so it must be rejected in favour of the sweeps; X+ is the
    projector-weighted sum and is basis-independent within each cluster."""
    for n, r in ((96, 9), (200, 12), (320, 20)):
        Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
        lam = -rng.random(n)
        top = np.concatenate([[7.0, 7.0 * (1 + 1e-10), 7.0 * (1 - 3e-12), 7.0 * (1 + 2e-11),
                               3.0, 3.0 * (1 + 1e-11), 3.0 * (1 - 1e-12), 1.5, 1.5 * (1 + 1e-10)],
                              0.5 + 0.4 * rng.random(r)])[:r]
        lam[:r] = top
        D = (Q * lam) @ Q.T
        S = orc.pack(0.5 * (D + D.T))
        P, lm = pk.aproj_psd(pk.SymMatrix(n, S), r)
        Pr, lr = orc.aproj_psd(S, n, r)
        assert rel(P.data, Pr) <= ITER_TOL
        assert lm == pytest.approx(lr, rel=1e-8, abs=1e-10)
        # X+ = Q_r diag(top) Q_r^T exactly (the construction), to the same tolerance
        exact = orc.pack((Q[:, :r] * top) @ Q[:, :r].T)
        assert rel(P.data, exact) <= ITER_TOL


# ---------------------------------------------------------------- full solves

@pytest.mark.parametrize("ci", range(5))
def test_small_lr_solves_match_reference(ci):
    d = load_golden("lr_small.npz")
    pre = f"c{ci}_"
    prob = problem_from_golden(d, pre)
    cfg = SolverConfig(eps_tol=1e-4, max_iter=400, initial_rank=int(d[pre + "r0"]),
                       window_ell=50, time_limit_s=1e9)
    res = pk.solve_lr_pd_sdp(prob, cfg)
    assert res.status.value == str(d[pre + "status"])
    assert res.iterations == int(d[pre + "iters"])
    assert [tuple(x) for x in res.rank_path] == [tuple(x) for x in d[pre + "rank_path"].tolist()]
    assert rel(res.X.data, d[pre + "X"]) <= ITER_TOL
    assert rel(res.y, d[pre + "y"]) <= ITER_TOL
    assert res.primal_objective == pytest.approx(float(d[pre + "pobj"]), rel=OBJ_TOL)
    assert res.dual_objective == pytest.approx(float(d[pre + "dobj"]), rel=OBJ_TOL)
    assert res.residual_scale == pytest.approx(float(d[pre + "scale"]), rel=1e-10)


def test_extrapolated_start_cuts_operator_applications():
    """The eigensolver starts each iteration from an extrapolation of the last
    eigenvector blocks (iterate.cuh, PDSDP_EXTRAP): same iterates as the
    oracle, but far fewer operator applications than the plain warm start
    needed on config 1 (15.9 per iteration; 8.3 measured with the
    extrapolation) -- guards against the start silently falling back."""
    from paper_1810_05231_b200.device import DeviceBatch
    from paper_1810_05231_b200.solver import operator_norm_on_device, run_lr_loop
    prob, cfg = workloads.config(0)
    batch = DeviceBatch([prob])
    alpha = cfg.alpha_safety / operator_norm_on_device(batch, 0, cfg.seed)
    o = run_lr_loop(batch, 0, prob, cfg, alpha)
    assert o.status.value == "optimal" and o.it.k == 1718
    assert o.eig_matvecs / o.it.k < 11.0
    batch.close()


def test_config1_end_to_end_matches_reference():
    d = load_golden("cfg1.npz")
    prob, cfg = workloads.config(0)
    for K in (1, 10, 100):
        res = pk.solve_lr_pd_sdp(prob, with_iters(cfg, K))
        assert res.iterations == K
        assert rel(res.X.data, d[f"X{K}"]) <= ITER_TOL
        assert rel(res.y, d[f"y{K}"]) <= ITER_TOL
        np.testing.assert_allclose(res.final_residuals, d[f"res{K}"], rtol=1e-8)
    hist = []
    res = pk.solve_lr_pd_sdp(prob, with_iters(cfg, cfg.max_iter, progress_every=1),
                             callback=lambda info: hist.append(tuple(info)))
    assert res.status.value == str(d["status"]) == "optimal"
    assert res.iterations == int(d["iters"]) == 1718
    assert [tuple(x) for x in res.rank_path] == [tuple(x) for x in d["rank_path"].tolist()]
    assert rel(res.X.data, d["X_final"]) <= ITER_TOL
    assert res.primal_objective == pytest.approx(float(d["pobj"]), rel=OBJ_TOL)
    assert res.dual_objective == pytest.approx(float(d["dobj"]), rel=OBJ_TOL)
    assert len(res.checkpoints) == len(d["checkpoints"])
    for c, (rk, obj) in zip(res.checkpoints, d["checkpoints"]):
        assert c.rank == int(rk) and c.objective == pytest.approx(obj, rel=OBJ_TOL)
    h = np.array(hist)
    np.testing.assert_allclose(h[:, 1:4], d["history"][:, 1:4], rtol=1e-6)
    np.testing.assert_allclose(h[:, 5], d["history"][:, 5], rtol=1e-8)


@pytest.mark.parametrize("idx,fname", [(4, "cfg5_sketch.npz"), (3, "cfg4_sketch.npz"),
                                       (1, "cfg2_sketch.npz"), (2, "cfg3_sketch.npz"),
                                       (2, "cfg3_stall_sketch.npz")])
def test_large_configs_fixed_K_sketches(idx, fname):
    """Configs 2-5 at the reference's full sizes, fixed K: y, diag(X), the
    sketch X z for a seeded z, ||X||_F, tr(CX) and the residuals."""
    d = load_golden(fname)
    prob, cfg = workloads.config(idx)
    z = np.random.default_rng(777).standard_normal(prob.n)
    # the power iteration stops on |s - sigma| <= 1e-10 s (problem.py:181), so
    # estimates agree to that order, not to rounding
    assert pk.estimate_operator_norm(prob, cfg.seed) == pytest.approx(float(d["opnorm"]), rel=1e-9)
    for K in d["Ks"].tolist():
        res = pk.solve_lr_pd_sdp(prob, with_iters(cfg, int(K)))
        Xd = res.X.to_dense()
        assert rel(res.y, d[f"y{K}"]) <= ITER_TOL
        assert rel(Xd @ z, d[f"Xz{K}"], floor=1e-4) <= ITER_TOL
        assert rel(np.diag(Xd), d[f"diag{K}"], floor=1e-4) <= ITER_TOL
        assert np.linalg.norm(Xd) == pytest.approx(float(d[f"fro{K}"]), rel=ITER_TOL)
        assert res.primal_objective == pytest.approx(float(d[f"pobj{K}"]), rel=OBJ_TOL, abs=1e-9)
        np.testing.assert_allclose(res.final_residuals, d[f"res{K}"], rtol=1e-7)


def test_oracle_parity_with_inequalities(rng):
    """Seeded random problems with inequality rows (exercises min(u/alpha, h)),
    against the oracle at fixed K."""
    for n, m, p, r0 in ((20, 10, 12, 1), (50, 20, 30, 3)):
        R = rng.standard_normal((n, n))
        C = pk.SymMatrix.from_dense(R @ R.T / n)
        rows = []
        for _ in range(m + p):
            ents = [(int(i), int(j), float(rng.standard_normal()))
                    for i, j in {tuple(sorted(rng.integers(0, n, 2))) for _ in range(4)}]
            rows.append(pk.SparseRow.from_matrix_entries(n, ents))
        prob = pk.SdpProblem(n=n, C=C, A=rows[:m], b=np.abs(rng.standard_normal(m)) + 0.5,
                             G=rows[m:], h=np.abs(rng.standard_normal(p)) + 0.2)
        cfg = SolverConfig(eps_tol=1e-6, max_iter=150, initial_rank=r0, window_ell=40)
        res = pk.solve_lr_pd_sdp(prob, cfg)
        ref = orc.solve_lr(prob, cfg)
        assert res.iterations == ref.iterations
        assert res.rank_path == ref.rank_path
        assert rel(res.X.data, ref.X) <= ITER_TOL
        assert rel(res.y, ref.y) <= ITER_TOL


def _rank_one_row(n, u, sig):
    return pk.SparseRow.from_matrix_entries(
        n, [(i, j, sig * u[i] * u[j]) for i in range(n) for j in range(i, n) if u[i] * u[j] != 0.0])


def test_dense_rank_one_rows_match_oracle(rng):
    """Dense constraint rows whose matrix is sig u u^T are applied through u on
    the device (equipartition's <11^T, X> = 0, BASELINE configs[2]); the
    results must not depend on that.  Covers sig = -1, a u with zeros (a dense
    sub-block), two such rows, and a dense rank-two row that stays in the CSR."""
    n = 90
    prob = workloads.equipartition_problem(n, 0.08, 5)
    cfg = SolverConfig(eps_tol=1e-4, max_iter=200, initial_rank=4)
    res = pk.solve_lr_pd_sdp(prob, cfg)
    ref = orc.solve_lr(prob, cfg)
    assert res.iterations == ref.iterations and res.rank_path == ref.rank_path
    assert rel(res.X.data, ref.X) <= ITER_TOL
    assert rel(res.y, ref.y) <= ITER_TOL
    np.testing.assert_allclose(res.final_residuals, ref.final_residuals, rtol=1e-7)

    g = workloads.random_graph(n, 0.1, 9, signed=True)
    C = pk.SymMatrix(n, workloads.laplacian_packed(g, -0.25))
    u1 = rng.standard_normal(n)
    u2 = np.where(np.arange(n) < n // 2, 1.0 + rng.random(n), 0.0)
    w1, w2 = rng.standard_normal(n), rng.standard_normal(n)
    rank2 = pk.SparseRow.from_matrix_entries(
        n, [(i, j, w1[i] * w1[j] - w2[i] * w2[j]) for i in range(n) for j in range(i, n)])
    rows = workloads.diag_pin_rows(n) + [_rank_one_row(n, u1, -1.0), _rank_one_row(n, u2, 1.0), rank2]
    prob = pk.SdpProblem(n=n, C=C, A=rows, b=np.concatenate([np.ones(n), [-0.5, 2.0, 0.1]]))
    cfg = SolverConfig(eps_tol=1e-6, max_iter=120, initial_rank=3, window_ell=60)
    res = pk.solve_lr_pd_sdp(prob, cfg)
    ref = orc.solve_lr(prob, cfg)
    assert res.iterations == ref.iterations and res.rank_path == ref.rank_path
    assert rel(res.X.data, ref.X) <= ITER_TOL
    assert rel(res.y, ref.y) <= ITER_TOL
    np.testing.assert_allclose(res.final_residuals, ref.final_residuals, rtol=1e-7)


# ---------------------------------------------------------------- edge cases

def test_oversized_steps_follow_reference():
    # reference test_pdhg.py:296-305 (alpha = 2/||M||) plus overflow regimes:
    # status and iteration count must match the oracle exactly.
    for n, a, K in ((2, None, 3000), (2, 1e100, 50), (40, 1e200, 50)):
        prob = pk.SdpProblem(n=n, C=pk.SymMatrix.from_dense(np.eye(n)),
                             A=[pk.SparseRow.from_matrix_entries(n, [(i, i, 1.0) for i in range(n)])],
                             b=np.array([1.0]))
        alpha = 2.0 / orc.op_norm(orc.stacked_csr(prob)) if a is None else a
        cfg = SolverConfig(alpha_override=alpha, max_iter=K, initial_rank=1)
        res = pk.solve_lr_pd_sdp(prob, cfg)
        ref = orc.solve_lr(prob, cfg)
        assert res.status.value == ref.status
        assert res.iterations == ref.iterations
        if np.all(np.isfinite(ref.y)):
            scale = max(np.abs(ref.y).max(), 1e-300)
            assert np.abs(res.y - ref.y).max() <= ITER_TOL * scale


def test_full_rank_and_tiny_problems():
    # r = n (no truncation, certificate vacuous) and n = 1
    prob = workloads.maxcut_problem(12, 0.5, 3, signed=True)
    cfg = SolverConfig(eps_tol=1e-5, max_iter=300, initial_rank=12)
    res = pk.solve_lr_pd_sdp(prob, cfg)
    ref = orc.solve_lr(prob, cfg)
    assert res.status.value == ref.status and res.iterations == ref.iterations
    assert rel(res.X.data, ref.X) <= ITER_TOL
    one = pk.SdpProblem(n=1, C=pk.SymMatrix(1, np.array([2.0])),
                        A=[pk.SparseRow(np.array([0]), np.array([1.0]))], b=np.array([3.0]))
    res = pk.solve_lr_pd_sdp(one, SolverConfig(max_iter=100))
    ref = orc.solve_lr(one, SolverConfig(max_iter=100))
    assert res.iterations == ref.iterations and res.status.value == ref.status
    assert res.primal_objective == pytest.approx(ref.primal_objective, rel=OBJ_TOL)


def test_target_rank_above_block_uses_positive_part():
    """Target ranks beyond the eigen block (the rank doubling of a stalled
    run, BASELINE configs[2]): only the positive eigenpairs plus a sentinel
    are computed; X+, y and the certificate decisions match the oracle, which
    uses dense eigh there (symmat.py:181-185)."""
    prob = workloads.equipartition_problem(150, 0.05, 2)
    for r0, K in ((100, 60), (150, 40), (70, 180)):   # X has 42 positive eigenpairs at k=180
        cfg = SolverConfig(eps_tol=1e-4, max_iter=K, initial_rank=r0, window_ell=50)
        res = pk.solve_lr_pd_sdp(prob, cfg)
        ref = orc.solve_lr(prob, cfg)
        assert res.iterations == ref.iterations and res.rank_path == ref.rank_path
        assert rel(res.X.data, ref.X) <= ITER_TOL
        assert rel(res.y, ref.y) <= ITER_TOL
        np.testing.assert_allclose(res.final_residuals, ref.final_residuals, rtol=1e-7)


def _unpack(n, v):
    iu, ju = np.triu_indices(n)
    w = np.array(v, dtype=float)
    w[iu != ju] /= np.sqrt(2.0)
    S = np.zeros((n, n))
    S[iu, ju] = w
    S[ju, iu] = w
    return S


@pytest.mark.parametrize("n,seed,ranks", [(100, 11, (60, 80, 100)), (300, 12, (100, 200, 300))])
def test_dense_eigensolver_aproj_matches_reference(n, seed, ranks):
    """aproj_psd where the reference takes dense eigh (2 (r+1) > n,
    symmat.py:181-185) or r + 1 exceeds the in-cluster eigen block: the device
    runs its full eigendecomposition (dense_path.cuh, one-sided Jacobi).
    Reference outputs: tests/golden/dense.npz (make_golden.py make_dense)."""
    from conftest import dense_case_matrix
    d = load_golden("dense.npz")
    S = pk.SymMatrix.from_dense(dense_case_matrix(n, seed))
    zs = np.random.default_rng(777).standard_normal((300, 4))[:n]
    for r in ranks:
        pre = f"ap_n{n}_r{r}_"
        P, lam = pk.aproj_psd(S, r)
        Pd = _unpack(n, P.data)
        assert lam == pytest.approx(float(d[pre + "lam"]), abs=1e-10)
        assert abs(np.linalg.norm(Pd) - float(d[pre + "fro"])) <= 1e-9 * float(d[pre + "fro"])
        assert rel(np.diag(Pd), d[pre + "diag"]) <= ITER_TOL
        assert rel(Pd @ zs, d[pre + "Pz"]) <= ITER_TOL
        if n == 100:
            assert rel(P.data, d[pre + "P"]) <= ITER_TOL


def test_dense_eigensolver_large_even_n_bulk_copy_rounds():
    """n = 3072 takes the Jacobi rounds whose rows move by TMA bulk copies
    (even n >= 3072); the full projection is checked against numpy's eigh, the
    reference's own dense method (symmat.py:158-161, 223-226)."""
    n = 3072
    rng = np.random.default_rng(31)
    R = rng.standard_normal((n, n))
    Sd = 0.5 * (R + R.T) / np.sqrt(n)
    P, lam = pk.aproj_psd(pk.SymMatrix.from_dense(Sd), n)
    w, V = np.linalg.eigh(Sd)
    assert lam == pytest.approx(w[0], abs=1e-9)
    keep = w > 0
    ref = (V[:, keep] * w[keep]) @ V[:, keep].T
    assert rel(_unpack(n, P.data), ref) <= ITER_TOL


def test_dense_eigensolver_blocked_rounds(monkeypatch):
    """The blocked Jacobi rounds (16-row blocks, in-CTA Gram eigensolve; taken
    for n >= 4096) forced at n = 300 / 515 (odd block count, ragged last
    block) against the reference's dense-path outputs and numpy eigh."""
    monkeypatch.setenv("PDSDP_DENSE_BLOCK_NMIN", "32")
    from conftest import dense_case_matrix
    d = load_golden("dense.npz")
    S = pk.SymMatrix.from_dense(dense_case_matrix(300, 12))
    zs = np.random.default_rng(777).standard_normal((300, 4))
    for r in (200, 300):
        P, lam = pk.aproj_psd(S, r)
        Pd = _unpack(300, P.data)
        assert lam == pytest.approx(float(d[f"ap_n300_r{r}_lam"]), abs=1e-10)
        assert rel(Pd @ zs, d[f"ap_n300_r{r}_Pz"]) <= ITER_TOL
    n = 515
    rng = np.random.default_rng(41)
    R = rng.standard_normal((n, n))
    Sd = 0.5 * (R + R.T) / np.sqrt(n)
    P, lam = pk.aproj_psd(pk.SymMatrix.from_dense(Sd), n)
    w, V = np.linalg.eigh(Sd)
    assert lam == pytest.approx(w[0], abs=1e-10)
    assert rel(_unpack(n, P.data), (V[:, w > 0] * w[w > 0]) @ V[:, w > 0].T) <= ITER_TOL


def test_exact_solver_above_block_limit_matches_reference():
    """solve_pd_sdp with n = 100 > PDSDP_BLOCK_MAX: every iteration is a full
    projection on the dense-iterate path (reference pdhg.py:221-288 with
    symmat.py:223-226); iterates at K = 1, 10, 50 and the solve to tolerance."""
    d = load_golden("dense.npz")
    prob = problem_from_golden(d, "pd_")
    for K in (1, 10, 50):
        res = pk.solve_pd_sdp(prob, SolverConfig(eps_tol=1e-4, max_iter=K, time_limit_s=1e9))
        assert res.iterations == K
        assert rel(res.X.data, d[f"pd_X{K}"]) <= ITER_TOL
        assert rel(res.y, d[f"pd_y{K}"]) <= ITER_TOL
        np.testing.assert_allclose(res.final_residuals, d[f"pd_res{K}"], rtol=1e-6)
    res = pk.solve_pd_sdp(prob, SolverConfig(eps_tol=1e-4, max_iter=5000, time_limit_s=1e9))
    assert res.status.value == str(d["pd_status"]) == "optimal"
    assert res.iterations == int(d["pd_iters"])
    assert res.rank_path == [(0, 100)]
    assert res.primal_objective == pytest.approx(float(d["pd_pobj"]), rel=OBJ_TOL)
    assert res.dual_objective == pytest.approx(float(d["pd_dobj"]), rel=OBJ_TOL)
    assert rel(res.X.data, d["pd_X"]) <= 1e-6


def test_rank_above_block_limit_continues_on_dense_path():
    """An LR run whose projection argument has more positive eigenvalues than
    an eigen block holds (the reference runs dense eigh there,
    symmat.py:181-185): the cluster kernel leaves that step unfinished and the
    solve continues on the dense-iterate path from the same (X_k, y_k)."""
    d = load_golden("dense.npz")
    # equipartition n = 150, r0 = 70: rank doubles to 140 / 150, X reaches 84 positive eigenpairs
    prob = workloads.equipartition_problem(150, 0.05, 2)
    cfg = SolverConfig(eps_tol=1e-4, max_iter=300, initial_rank=70, window_ell=50, time_limit_s=1e9)
    res = pk.solve_lr_pd_sdp(prob, cfg)
    assert res.status.value == str(d["lr_status"])
    assert res.iterations == int(d["lr_iters"])
    assert res.rank_path == [tuple(int(v) for v in row) for row in d["lr_rank_path"]]
    assert int(d["lr_npos"]) > 64
    assert rel(res.X.data, d["lr_X"]) <= ITER_TOL
    assert rel(res.y, d["lr_y"]) <= ITER_TOL
    np.testing.assert_allclose(res.final_residuals, d["lr_res"], rtol=1e-6)
    assert res.primal_objective == pytest.approx(float(d["lr_pobj"]), rel=OBJ_TOL)
    # Max-Cut n = 200, r0 = 80: S_1 = alpha L / 4 has ~n positive eigenvalues at the first step
    prob = workloads.maxcut_problem(200, 0.1, 0, signed=False)
    res = pk.solve_lr_pd_sdp(prob, SolverConfig(initial_rank=80, max_iter=2, time_limit_s=1e9))
    assert res.iterations == 2
    assert rel(res.X.data, d["mc_X"]) <= ITER_TOL
    assert rel(res.y, d["mc_y"]) <= ITER_TOL
    np.testing.assert_allclose(res.final_residuals, d["mc_res"], rtol=1e-6)


# ------------------------------------------------- solves to tolerance, full size

FULL_CASES = [("cfg2_full.npz", 1, 0), ("cfg5s0_full.npz", 4, 0), ("cfg5s1_full.npz", 4, 1),
              ("cfg5s2_full.npz", 4, 2), ("cfg5s3_full.npz", 4, 3), ("cfg4_full.npz", 3, 0)]


@pytest.mark.parametrize("fname,idx,seed", FULL_CASES)
def test_solve_to_tolerance_matches_reference(fname, idx, seed, capsys):
    """BASELINE configs 2, 4, 5 solved to the 1e-4 rule on the GPU against the
    UNMODIFIED reference run to tolerance on the same seeded input
    (tests/golden/make_golden.py --full: status, stop iteration, rank path,
    checkpoints, objectives, final residuals, final X as eigen-factors).
    North-star bar: objective within 1e-5 relative, the same 1e-4 stopping
    rule met.  Long solves are chaotic in the stall-triggered rank-doubling
    times (eigensolver differences at ARPACK's own 1e-12 move them), so the
    iteration counts are compared with a tolerance and the delta is printed;
    the sequence of ranks must be identical."""
    d = load_golden(fname)
    prob, cfg = workloads.config(idx, seed)
    res = pk.solve_lr_pd_sdp(prob, cfg)
    assert res.status.value == str(d["status"]) == "optimal"
    ref_iters = int(d["iters"])
    ref_path = [tuple(int(v) for v in row) for row in d["rank_path"]]
    # config 4 (idx 3) is chaotic at rounding level in the reference itself
    # (profiles/r02_cfg4_reference_chaos_arpack_seed.txt): its rank sequence is
    # reported, not required; every other config must reproduce it
    chaotic = idx == 3
    if not chaotic:
        assert [r for _, r in res.rank_path] == [r for _, r in ref_path]
    assert res.residual_scale == pytest.approx(float(d["scale"]), rel=1e-9)
    # the same stopping rule met by both (lowrank.py:153-161)
    assert res.final_residuals[2] <= cfg.eps_tol * res.residual_scale
    assert float(d["res_final"][2]) <= cfg.eps_tol * float(d["scale"])
    assert res.primal_objective == pytest.approx(float(d["pobj"]), rel=OBJ_TOL)
    same_path = res.rank_path == ref_path
    if same_path:
        assert res.dual_objective == pytest.approx(float(d["dobj"]), rel=OBJ_TOL)
    else:
        # different rank-doubling times = a different trajectory to the same
        # optimum: the dual objective of either run is only as accurate as its
        # duality gap at the 1e-4 stop (config 4: gap 1.0e-3, difference 1.3e-4)
        gap = abs(float(d["pobj"]) - float(d["dobj"]))
        assert abs(res.dual_objective - float(d["dobj"])) <= gap
    if not chaotic:
        assert len(res.checkpoints) == len(d["checkpoints"])
        for c, (rk, obj) in zip(res.checkpoints, d["checkpoints"]):
            assert c.rank == int(rk) and c.objective == pytest.approx(obj, rel=1e-4)
        assert abs(res.iterations - ref_iters) <= 0.05 * ref_iters
    else:
        assert res.checkpoints[-1].objective == pytest.approx(float(d["checkpoints"][-1][1]), rel=OBJ_TOL)
        assert abs(res.iterations - ref_iters) <= 0.25 * ref_iters
    # exact rel-Frobenius distance of the final iterates (reference X = V diag(lam) V^T)
    V, lam = d["X_V"], d["X_lam"]
    Xg = res.X.to_dense()
    err = np.linalg.norm(Xg - (V * lam) @ V.T) / float(d["X_fro"])
    yerr = rel(res.y, d["y_final"])
    with capsys.disabled():
        print(f"\n[{fname}] iterations {res.iterations} vs reference {ref_iters} (delta {res.iterations - ref_iters}), "
              f"rank path {res.rank_path} vs {ref_path}, pobj rel diff "
              f"{abs(res.primal_objective - float(d['pobj'])) / abs(float(d['pobj'])):.2e}, dobj rel diff "
              f"{abs(res.dual_objective - float(d['dobj'])) / abs(float(d['dobj'])):.2e}, "
              f"final X rel-Frobenius diff {err:.2e}, y rel diff {yerr:.2e}")
    if same_path and res.iterations == ref_iters:
        assert err <= 1e-6 and yerr <= 1e-6      # same trajectory: only eigensolver-level differences
    else:
        assert err <= 5e-3                       # both within the 1e-4 rule of the same optimum


def test_time_limit_and_max_iter_status():
    prob, cfg = workloads.config(0)
    res = pk.solve_lr_pd_sdp(prob, with_iters(cfg, 7))
    assert res.status.value == "max_iterations" and res.iterations == 7
    res = pk.solve_lr_pd_sdp(prob, with_iters(cfg, 100000, time_limit_s=1e-9))
    assert res.status.value == "time_limit" and res.iterations == 1


def test_batched_solve_matches_single_instance_solves():
    """config-5 style batch: independent instances solved together give the
    same iterations, rank paths and iterates as one-at-a-time solves."""
    probs = [workloads.maxcut_problem(100, 0.1, seed, signed=True) for seed in range(4)]
    cfg = SolverConfig(eps_tol=1e-4, max_iter=600, initial_rank=2, window_ell=100)
    batch = pk.solve_lr_pd_sdp_batch(probs, cfg)
    for p, rb in zip(probs, batch):
        rs = pk.solve_lr_pd_sdp(p, cfg)
        ro = orc.solve_lr(p, cfg)
        assert rb.status == rs.status and rb.iterations == rs.iterations == ro.iterations
        assert rb.rank_path == rs.rank_path == ro.rank_path
        assert rel(rb.X.data, rs.X.data) <= 1e-12
        assert rel(rb.X.data, ro.X) <= ITER_TOL


def test_batch_with_instance_switching_to_dense_path():
    """A batch in which one instance leaves the cluster kernel for the
    dense-iterate path mid-run (more positive eigenvalues than an eigen block
    holds) while the others stay on it: every instance matches its own
    single-instance solve, so the slot scheduler does not mix the two modes."""
    probs = [workloads.maxcut_problem(60, 0.15, 3, signed=True),
             workloads.equipartition_problem(150, 0.05, 2),
             workloads.maxcut_problem(80, 0.1, 4, signed=True)]
    cfg = SolverConfig(eps_tol=1e-4, max_iter=300, initial_rank=70, window_ell=50, time_limit_s=1e9)
    batch = pk.solve_lr_pd_sdp_batch(probs, cfg)     # initial_rank is clipped to n per problem
    for p, rb in zip(probs, batch):
        rs = pk.solve_lr_pd_sdp(p, cfg)
        assert rb.status == rs.status and rb.iterations == rs.iterations
        assert rb.rank_path == rs.rank_path
        assert rel(rb.X.data, rs.X.data) <= 1e-12
        assert rel(rb.y, rs.y) <= 1e-12


def test_large_batch_runs_on_half_size_clusters():
    """A batch with more instances than clusters can be resident is laid out
    on clusters of half the default size (pdsdp_batch_create); the instances
    still follow their single-solve trajectories (rounding-level differences
    of the cluster reductions only)."""
    from paper_1810_05231_b200.device import DeviceBatch
    n = 260                                   # 3 CTAs of 128 rows -> clusters of 4 by default
    few = [workloads.maxcut_problem(n, 0.05, s, signed=True) for s in range(2)]
    b_few = DeviceBatch(few)
    c_default = b_few.info(0)["cluster"]
    b_few.close()
    assert c_default == 4
    # at most 148 / 4 = 37 clusters of 4 CTAs fit the device
    probs = [workloads.maxcut_problem(n, 0.05, s, signed=True) for s in range(40)]
    cfg = SolverConfig(eps_tol=1e-4, max_iter=150, initial_rank=3, window_ell=60)
    b_many = DeviceBatch(probs)
    assert b_many.info(0)["cluster"] == c_default // 2
    b_many.close()
    batch = pk.solve_lr_pd_sdp_batch(probs, cfg)
    assert len(batch) == len(probs)
    for p, rb in list(zip(probs, batch))[:3]:
        rs = pk.solve_lr_pd_sdp(p, cfg)
        assert rb.status == rs.status and rb.iterations == rs.iterations and rb.rank_path == rs.rank_path
        assert rel(rb.X.data, rs.X.data) <= 1e-9
        assert rel(rb.y, rs.y) <= 1e-9


# ------------------------------------------- factored vs entrywise residual

@pytest.mark.parametrize("ci,K,r", [(0, 300, 5), (1, 40, 10), (3, 30, 1), (4, 40, 1)])
def test_dense_residual_factored_matches_entrywise(ci, K, r):
    """The iteration kernel evaluates ||dX/alpha||_F^2 (reference
    pdhg.py:198-208) in factored form from V^T F and F_perp^T F_perp; the
    verification kernel evaluates it entry by entry over the upper triangle.
    They must agree to rounding at every step (1e-9 relative)."""
    from paper_1810_05231_b200.device import DeviceBatch, OUT_DENSE, OUT_DENSE_EXACT, OUT_DONE
    from paper_1810_05231_b200.solver import operator_norm_on_device
    prob, cfg = workloads.config(ci)
    b = DeviceBatch([prob])
    alpha = cfg.alpha_safety / operator_norm_on_device(b, 0, 0)
    b.set_alpha(0, alpha)
    b.reset(0, 0.0)
    b.set_verify_residual(True)
    ypar, checked = 0, 0
    for k in range(K):
        o = b.iterate([0], [r], [ypar])[0]
        ypar ^= 1
        assert o[OUT_DONE] == 1.0
        ex, fa = o[OUT_DENSE_EXACT], o[OUT_DENSE]
        assert np.isfinite(ex)
        assert abs(fa - ex) <= 1e-9 * max(abs(ex), 1e-300) + 1e-24, (k, fa, ex)
        checked += 1
    b.close()
    assert checked == K


# ------------------------------------------------ exact PD-SDP

@pytest.mark.parametrize("ci", range(4))
def test_exact_pd_sdp_matches_reference(ci):
    """solve_pd_sdp (reference pdhg.py:221-288, full projection) against the
    reference's own solves: iterates at K = 1, 10 and the full run (status,
    iteration count, iterates, objectives)."""
    d = load_golden("pd_small.npz")
    pre = f"c{ci}_"
    prob = problem_from_golden(d, pre)
    for K in (1, 10):
        res = pk.solve_pd_sdp(prob, SolverConfig(eps_tol=1e-4, max_iter=K, time_limit_s=1e9))
        assert res.iterations == K
        # an iterate that is zero up to rounding (the MIMO objective is PSD, so
        # proj_psd(-alpha C) = 0; LAPACK leaves ~1e-16 eigenvalues, the device
        # clips them) is compared absolutely against the floor
        assert rel(res.X.data, d[pre + f"X{K}"], floor=1e-6) <= ITER_TOL
        assert rel(res.y, d[pre + f"y{K}"]) <= ITER_TOL
        np.testing.assert_allclose(res.final_residuals, d[pre + f"res{K}"], rtol=1e-7, atol=1e-12)
    res = pk.solve_pd_sdp(prob, SolverConfig(eps_tol=1e-4, max_iter=3000, time_limit_s=1e9))
    assert res.status.value == str(d[pre + "status"])
    assert res.iterations == int(d[pre + "iters"])
    assert res.rank_path == [(0, prob.n)] and res.checkpoints == []
    assert rel(res.X.data, d[pre + "X"]) <= ITER_TOL
    assert rel(res.y, d[pre + "y"]) <= ITER_TOL
    assert res.primal_objective == pytest.approx(float(d[pre + "pobj"]), rel=OBJ_TOL, abs=1e-9)
    assert res.dual_objective == pytest.approx(float(d[pre + "dobj"]), rel=OBJ_TOL, abs=1e-9)


# ------------------------------------ inequality-heavy MIMO

@pytest.mark.parametrize("ci", range(2))
def test_mimo_lr_matches_reference(ci):
    """LR-PD-SDP on the reference's MIMO relaxation (instances.gen_mimo: n+1
    pins and 2 per off-diagonal box inequality rows, i.e. the proj_box branch
    of the dual step on n(n+1) rows)."""
    d = load_golden("mimo.npz")
    pre = f"c{ci}_"
    prob = problem_from_golden(d, pre)
    K = int(d[pre + "K"])
    res = pk.solve_lr_pd_sdp(prob, SolverConfig(eps_tol=1e-4, max_iter=K, initial_rank=1, window_ell=50,
                                                time_limit_s=1e9))
    assert res.status.value == str(d[pre + "status"])
    assert res.iterations == int(d[pre + "iters"])
    assert [tuple(x) for x in res.rank_path] == [tuple(x) for x in d[pre + "rank_path"].tolist()]
    assert rel(res.X.data, d[pre + "X"]) <= ITER_TOL
    assert rel(res.y, d[pre + "y"]) <= ITER_TOL
    assert res.primal_objective == pytest.approx(float(d[pre + "pobj"]), rel=OBJ_TOL)


# --------------------------------------- check_solution

def test_check_solution_matches_reference():
    """check_solution (reference problem.py:213-240) with A(X) and the
    minimum eigenvalue on the device, against the reference's reports."""
    d = load_golden("check.npz")
    keys = sorted({k.split("_")[0] + "_" + k.split("_")[1] for k in d.files if k.startswith("k")})
    assert keys
    for q in keys:
        q = q + "_"
        prob = problem_from_golden(d, q)
        rep = pk.check_solution(prob, pk.SymMatrix(prob.n, d[q + "X"]), d[q + "yv"])
        ref = d[q + "report"]
        got = np.array([rep.primal_objective, rep.dual_objective, rep.equality_violation,
                        rep.inequality_violation, rep.min_eigenvalue, rep.duality_gap])
        scale = max(1.0, float(np.abs(d[q + "X"]).max()))
        np.testing.assert_allclose(got[[0, 1, 5]], ref[[0, 1, 5]], rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(got[[2, 3]], ref[[2, 3]], rtol=1e-10, atol=1e-12)
        assert abs(got[4] - ref[4]) <= 1e-8 * scale, (q, got[4], ref[4])
        assert rep.max_violation() == pytest.approx(max(ref[2], ref[3], -min(ref[4], 0.0)), rel=1e-6, abs=1e-8 * scale)


# ---------------------------------------------------------------- reference-typed inputs

class _RefLayoutSym:
    """Stand-in with the reference SymMatrix's layout (``symmat.py:104-113``)."""
    def __init__(self, n, data):
        self.n, self.data = n, data


class _RefLayoutRow:
    def __init__(self, indices, values):
        self.indices, self.values = indices, values


class _RefLayoutProblem:
    """Stand-in with the fields of the reference's ``SdpProblem``
    (``problem.py:74-87``) and none of this package's (no ``_device_cache``,
    no ``stacked_arrays``): what ``cli._solve_one`` would hand over.  The real
    reference types are exercised in tests/test_dropin_cpu.py (the reference
    tree does not exist on the GPU box)."""
    def __init__(self, prob):
        self.n = prob.n
        self.C = _RefLayoutSym(prob.n, prob.C.data.copy())
        self.A = [_RefLayoutRow(r.indices.copy(), r.values.copy()) for r in prob.A]
        self.b = prob.b.copy()
        self.G = [_RefLayoutRow(r.indices.copy(), r.values.copy()) for r in prob.G]
        self.h = prob.h.copy()
        self.name = "ref-layout"
        self.objective_sign = 1.0


def test_reference_layout_problem_solves_identically():
    d = load_golden("lr_small.npz")
    pre = "c1_"
    prob = problem_from_golden(d, pre)
    cfg = SolverConfig(eps_tol=1e-4, max_iter=400, initial_rank=int(d[pre + "r0"]),
                       window_ell=50, time_limit_s=1e9)
    dup = _RefLayoutProblem(prob)
    res = pk.solve_lr_pd_sdp(dup, cfg)
    assert res.status.value == str(d[pre + "status"]) and res.iterations == int(d[pre + "iters"])
    assert rel(res.X.data, d[pre + "X"]) <= ITER_TOL and rel(res.y, d[pre + "y"]) <= ITER_TOL
    # op-level entry points and the report take the same object
    own = pk.solve_lr_pd_sdp(prob, cfg)
    assert np.array_equal(own.X.data, res.X.data) and np.array_equal(own.y, res.y)
    np.testing.assert_array_equal(pk.apply_M(dup, res.X), pk.apply_M(prob, res.X))
    np.testing.assert_array_equal(pk.apply_M_adjoint(dup, res.y).data, pk.apply_M_adjoint(prob, res.y).data)
    assert pk.estimate_operator_norm(dup, 0) == pk.estimate_operator_norm(prob, 0)
    assert pk.check_solution(dup, res.X, res.y) == pk.check_solution(prob, res.X, res.y)
    assert not hasattr(dup, "_device_cache")
