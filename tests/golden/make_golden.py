"""Generate golden fixtures by running the REFERENCE implementation itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py [--big]

It imports the unmodified reference package from /root/reference/pkg/src and
records, for seeded inputs built with ``paper_1810_05231_b200.workloads``:

* ``ops_small.npz``   — operator-level known answers (apply_M, adjoint,
  operator norm, aproj_psd incl. the ARPACK path, dual step, residuals) on
  random problems shaped like the reference's own ``conftest.random_problem``;
* ``lr_small.npz``    — full LR-PD-SDP solves of small problems (with
  inequalities, so the box projection branch is exercised);
* ``pd_small.npz``    — exact PD-SDP solves (``solve_pd_sdp``, full projection)
  of small problems incl. a MIMO relaxation, iterates at K = 1, 10;
* ``mimo.npz``        — LR-PD-SDP on MIMO relaxations (inequality-heavy);
* ``check.npz``       — ``check_solution`` reports;
* ``io.npz``          — SDPA / extended-JSON parses and rewrites, parse errors,
  a solution document (reference ``io.py``);
* ``cfg1.npz``        — BASELINE config 1 (n=100 Max-Cut): iterates at
  K = 1, 10, 100 and at the stop iteration, per-iteration residual history,
  final objective / rank path / checkpoints;
* ``cfgN_sketch.npz`` (``--big``) — configs 2-5 at small K: y, lambda_{r+1},
  residuals, tr(CX), ||X||_F and the sketch X @ z for a seeded z (sketches
  keep the fixtures small while pinning the full n x n iterate).

* ``dense.npz``       — where the reference runs dense eigh: aproj_psd at n = 100 /
  300 with large r, exact PD-SDP at n = 100, an LR run whose rank crosses 64;
* ``cfgN_full.npz`` / ``cfg5sK_full.npz`` (``--full cfg2,cfg4,cfg5s0,...``; hours of
  CPU each) — the UNMODIFIED reference run to tolerance: status, stop iteration,
  rank path, checkpoints, objectives, residuals, y, the final X as eigen-factors,
  the progress history every 100 iterations;
* ``cfg3_stall_sketch.npz`` (``--full cfg3_stall``) — config 3 at K = 510, past its
  first stall-triggered rank doubling.

The reference crashes on config 4 iteration 1 (ArpackError -9, SURVEY.md §8c
quirk 1); for that config only the harness wraps ``truncated_eigen`` with the
reference's own dense fallback (``symmat.py:200-207``).
"""

from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import pdsdp  # noqa: E402  (the reference)
import pdsdp.lowrank as ref_lowrank  # noqa: E402
import pdsdp.symmat as ref_symmat  # noqa: E402
from pdsdp import SdpProblem as RProblem, SparseRow as RRow, SymMatrix as RSym  # noqa: E402
from scipy.sparse.linalg import ArpackError  # noqa: E402

from paper_1810_05231_b200 import workloads  # noqa: E402
sys.path.insert(0, os.path.dirname(HERE))
from conftest import dense_case_matrix  # noqa: E402  (seeded matrices shared with the GPU tests)

SKETCH_SEED = 777


def to_ref(prob):
    return RProblem(
        n=prob.n, C=RSym(prob.n, prob.C.data.copy()),
        A=[RRow(r.indices, r.values) for r in prob.A], b=prob.b.copy(),
        G=[RRow(r.indices, r.values) for r in prob.G], h=prob.h.copy(),
        name=prob.name, objective_sign=prob.objective_sign)


def to_ref_cfg(cfg, **over):
    d = dict(cfg.__dict__)
    d.update(over)
    return pdsdp.SolverConfig(**d)


class LambdaRecorder:
    """Wraps lowrank.aproj_psd to record lambda_{r+1} per iteration."""

    def __init__(self):
        self.values = []
        self.orig = ref_lowrank.aproj_psd

    def __enter__(self):
        def wrapped(S, r):
            out = self.orig(S, r)
            self.values.append(out[1])
            return out
        ref_lowrank.aproj_psd = wrapped
        return self

    def __exit__(self, *a):
        ref_lowrank.aproj_psd = self.orig


class ArpackErrorFallback:
    def __enter__(self):
        self.orig = ref_symmat.truncated_eigen

        def wrapped(S, r):
            try:
                return self.orig(S, r)
            except ArpackError:
                full = ref_symmat.full_eigen(S)
                return ref_symmat.EigenDecomposition(
                    full.values[:r].copy(), full.vectors[:, :r].copy(), r)
        ref_symmat.truncated_eigen = wrapped
        return self

    def __exit__(self, *a):
        ref_symmat.truncated_eigen = self.orig


def random_problem(n, m, p, rng, nnz=4):
    """Same construction as the reference's conftest.random_problem."""
    def entries():
        pairs = [(i, j) for i in range(n) for j in range(i, n)]
        idx = rng.choice(len(pairs), size=min(nnz, len(pairs)), replace=False)
        return [(pairs[k][0], pairs[k][1], float(rng.standard_normal())) for k in idx]
    R = rng.standard_normal((n, n))
    C = 0.5 * (R + R.T)
    A = [pdsdp.SparseRow.from_matrix_entries(n, entries()) for _ in range(m)]
    G = [pdsdp.SparseRow.from_matrix_entries(n, entries()) for _ in range(p)]
    return pdsdp.SdpProblem(n=n, C=pdsdp.SymMatrix.from_dense(C), A=A,
                            b=rng.standard_normal(m), G=G, h=rng.standard_normal(p))


def flatten_problem(prefix, prob, out):
    out[prefix + "n"] = prob.n
    out[prefix + "C"] = prob.C.data
    rows = list(prob.A) + list(prob.G)
    out[prefix + "indptr"] = np.cumsum([0] + [r.indices.size for r in rows])
    out[prefix + "idx"] = np.concatenate([r.indices for r in rows])
    out[prefix + "val"] = np.concatenate([r.values for r in rows])
    out[prefix + "b"] = prob.b
    out[prefix + "h"] = prob.h


def make_ops_small(path):
    rng = np.random.default_rng(12345)
    out = {}
    cases = [(6, 4, 2), (9, 5, 3), (12, 7, 0), (40, 12, 6), (64, 20, 4)]
    for ci, (n, m, p) in enumerate(cases):
        prob = random_problem(n, m, p, rng, nnz=5)
        pre = f"c{ci}_"
        flatten_problem(pre, prob, out)
        X = pdsdp.SymMatrix.from_dense((lambda R: R @ R.T)(rng.standard_normal((n, 3))))
        y = rng.standard_normal(m + p)
        out[pre + "X"] = X.data
        out[pre + "y"] = y
        out[pre + "MX"] = pdsdp.apply_M(prob, X)
        out[pre + "MTy"] = pdsdp.apply_M_adjoint(prob, y).data
        out[pre + "opnorm"] = pdsdp.estimate_operator_norm(prob, 0)
        S = pdsdp.SymMatrix.from_dense((lambda R: 0.5 * (R + R.T))(rng.standard_normal((n, n))))
        out[pre + "S"] = S.data
        for r in (1, 3, n // 2, n):
            P, lam = pdsdp.aproj_psd(S, r)
            out[pre + f"aproj{r}"] = P.data
            out[pre + f"aproj{r}_lam"] = lam
        e = pdsdp.truncated_eigen(S, min(5, n))
        out[pre + "teig_vals"] = e.values
        alpha = 0.37
        Xn = pdsdp.SymMatrix.from_dense((lambda R: R @ R.T)(rng.standard_normal((n, 2))))
        from pdsdp.pdhg import IterateState, dual_step, residuals
        from collections import deque
        yn = dual_step(prob, y, Xn, X, alpha)
        out[pre + "Xn"] = Xn.data
        out[pre + "dual"] = yn
        st = IterateState(Xn, X, yn, y, 1, deque())
        out[pre + "resid"] = np.array(residuals(st, alpha, prob))
    np.savez_compressed(path, **out)


def make_lr_small(path):
    rng = np.random.default_rng(2024)
    out = {}
    specs = [(8, 5, 0, 1), (10, 6, 4, 1), (16, 8, 6, 2), (36, 20, 10, 2), (48, 48, 0, 3)]
    for ci, (n, m, p, r0) in enumerate(specs):
        if ci == 4:   # Max-Cut shaped (diag pins), exercises the ARPACK path
            prob = to_ref(workloads.maxcut_problem(n, 0.2, 11, signed=True))
        else:
            prob = random_problem(n, m, p, rng, nnz=4)
            # make it well-posed: objective PSD-ish so the LR solve converges
            R = rng.standard_normal((n, n))
            prob = pdsdp.SdpProblem(n=n, C=pdsdp.SymMatrix.from_dense(R @ R.T / n),
                                    A=prob.A, b=np.abs(prob.b) + 0.5, G=prob.G,
                                    h=np.abs(prob.h) + 0.5)
        pre = f"c{ci}_"
        flatten_problem(pre, prob, out)
        cfg = pdsdp.SolverConfig(eps_tol=1e-4, max_iter=400, initial_rank=r0, window_ell=50,
                                 time_limit_s=1e9)
        with LambdaRecorder() as rec:
            res = pdsdp.solve_lr_pd_sdp(prob, cfg)
        out[pre + "r0"] = r0
        out[pre + "status"] = res.status.value
        out[pre + "iters"] = res.iterations
        out[pre + "X"] = res.X.data
        out[pre + "y"] = res.y
        out[pre + "pobj"] = res.primal_objective
        out[pre + "dobj"] = res.dual_objective
        out[pre + "res"] = np.array(res.final_residuals)
        out[pre + "rank_path"] = np.array(res.rank_path)
        out[pre + "lam"] = np.array(rec.values)
        out[pre + "scale"] = res.residual_scale
    np.savez_compressed(path, **out)


def make_cfg1(path):
    prob, cfg = workloads.config(0)
    rp = to_ref(prob)
    out = {}
    flatten_problem("", rp, out)
    for K in (1, 10, 100):
        with LambdaRecorder() as rec:
            res = pdsdp.solve_lr_pd_sdp(rp, to_ref_cfg(cfg, max_iter=K))
        out[f"X{K}"] = res.X.data
        out[f"y{K}"] = res.y
        out[f"lam{K}"] = rec.values[-1]
        out[f"res{K}"] = np.array(res.final_residuals)
    hist = []
    t0 = time.perf_counter()
    with LambdaRecorder() as rec:
        res = pdsdp.solve_lr_pd_sdp(rp, to_ref_cfg(cfg, progress_every=1),
                                    callback=lambda info: hist.append(tuple(info)))
    out["wall"] = time.perf_counter() - t0
    out["status"] = res.status.value
    out["iters"] = res.iterations
    out["X_final"] = res.X.data
    out["y_final"] = res.y
    out["pobj"] = res.primal_objective
    out["dobj"] = res.dual_objective
    out["res_final"] = np.array(res.final_residuals)
    out["rank_path"] = np.array(res.rank_path)
    out["checkpoints"] = np.array([(c.rank, c.objective) for c in res.checkpoints])
    out["scale"] = res.residual_scale
    out["history"] = np.array(hist)
    out["lam_hist"] = np.array(rec.values)
    np.savez_compressed(path, **out)
    print("cfg1", res.status, res.iterations, res.primal_objective, out["wall"])


def make_sketch(path, idx, Ks):
    prob, cfg = workloads.config(idx)
    t0 = time.perf_counter()
    rp = to_ref(prob)
    out = {"n": prob.n}
    z = np.random.default_rng(SKETCH_SEED).standard_normal(prob.n)
    guard = ArpackErrorFallback() if idx == 3 else None
    if guard:
        guard.__enter__()
    try:
        alpha = None
        for K in Ks:
            with LambdaRecorder() as rec:
                res = pdsdp.solve_lr_pd_sdp(rp, to_ref_cfg(cfg, max_iter=K))
            Xd = res.X.to_dense()
            out[f"y{K}"] = res.y
            out[f"lam{K}"] = np.array(rec.values)
            out[f"res{K}"] = np.array(res.final_residuals)
            out[f"pobj{K}"] = res.primal_objective
            out[f"fro{K}"] = np.linalg.norm(Xd)
            out[f"Xz{K}"] = Xd @ z
            out[f"diag{K}"] = np.diag(Xd).copy()
            out[f"rank_path{K}"] = np.array(res.rank_path)
            print(f"cfg{idx + 1} K={K} {time.perf_counter() - t0:.1f}s res={res.final_residuals}")
        from pdsdp.problem import estimate_operator_norm
        out["opnorm"] = estimate_operator_norm(rp, cfg.seed)
    finally:
        if guard:
            guard.__exit__()
    out["Ks"] = np.array(Ks)
    np.savez_compressed(path, **out)


def make_full(path, idx, seed=0):
    """Run the UNMODIFIED reference to tolerance on BASELINE config idx
    (0-based) and record what pins an end-to-end comparison: status, stop
    iteration, rank path, checkpoints, final objectives / residuals, y, the
    final X as eigen-factors (exact rank <= r, so V diag(lam) V^T reproduces
    the packed X to rounding) and the progress history every 100 iterations.
    Hours of CPU for configs 2 / 4; progress goes to stdout."""
    prob, cfg = workloads.config(idx, seed)
    rp = to_ref(prob)
    hist = []
    t0 = time.perf_counter()

    def cb(info):
        hist.append(tuple(info))
        if info.k % 1000 == 0:
            print(f"cfg{idx + 1} s{seed} k={info.k} eps_c={info.eps_comb:.3e} r={info.rank} "
                  f"obj={info.objective:.9g} t={time.perf_counter() - t0:.0f}s", flush=True)

    guard = ArpackErrorFallback() if idx == 3 else None
    if guard:
        guard.__enter__()
    try:
        with LambdaRecorder() as rec:
            res = pdsdp.solve_lr_pd_sdp(rp, to_ref_cfg(cfg, progress_every=100), callback=cb)
    finally:
        if guard:
            guard.__exit__()
    wall = time.perf_counter() - t0
    Xd = res.X.to_dense()
    w, V = np.linalg.eigh(Xd)
    keep = np.abs(w) > 1e-13 * max(np.abs(w).max(), 1e-300)
    w, V = w[keep][::-1], V[:, keep][:, ::-1]
    recon = (V * w) @ V.T
    out = {
        "n": prob.n, "seed": seed, "status": res.status.value, "iters": res.iterations,
        "pobj": res.primal_objective, "dobj": res.dual_objective,
        "res_final": np.array(res.final_residuals), "scale": res.residual_scale,
        "rank_path": np.array(res.rank_path),
        "checkpoints": np.array([(c.rank, c.objective) for c in res.checkpoints]),
        "y_final": res.y, "X_lam": w, "X_V": V,
        "X_fro": np.linalg.norm(Xd), "X_recon_err": np.linalg.norm(recon - Xd),
        "history": np.array(hist), "lam_last": rec.values[-1],
        "lam_at_rank_change": np.array([rec.values[k - 1] for k, _ in res.rank_path[1:]]),
        "wall": wall, "threads": os.environ.get("OMP_NUM_THREADS", ""),
    }
    np.savez_compressed(path, **out)
    print(f"cfg{idx + 1} s{seed} FULL {res.status} iters={res.iterations} pobj={res.primal_objective!r} "
          f"dobj={res.dual_objective!r} rank_path={res.rank_path} wall={wall:.0f}s "
          f"recon_err={out['X_recon_err']:.2e}", flush=True)


def _well_posed(prob, rng):
    """The reference conftest's random problem made feasible-ish (PSD
    objective, positive right-hand sides) so that solves converge."""
    n = prob.n
    R = rng.standard_normal((n, n))
    return pdsdp.SdpProblem(n=n, C=pdsdp.SymMatrix.from_dense(R @ R.T / n), A=prob.A,
                            b=np.abs(prob.b) + 0.5, G=prob.G, h=np.abs(prob.h) + 0.5)


def _mimo(n, sigma, seed):
    from pdsdp.instances import gen_mimo, random_mimo_instance
    return gen_mimo(random_mimo_instance(n, sigma, seed))


def make_pd_small(path):
    """Exact PD-SDP (reference pdhg.solve_pd_sdp, full projection) on small
    problems: random with inequalities, Max-Cut shaped, MIMO (box
    inequalities on every off-diagonal entry).  Iterates at K = 1, 10 and
    the full solve."""
    rng = np.random.default_rng(77)
    out = {}
    probs = [_well_posed(random_problem(10, 6, 4, rng, nnz=4), rng),
             to_ref(workloads.maxcut_problem(30, 0.2, 5, signed=True)),
             _mimo(12, 0.3, 3),
             _well_posed(random_problem(48, 20, 8, rng, nnz=4), rng)]
    for ci, prob in enumerate(probs):
        pre = f"c{ci}_"
        flatten_problem(pre, prob, out)
        for K in (1, 10):
            cfg = pdsdp.SolverConfig(eps_tol=1e-4, max_iter=K, time_limit_s=1e9)
            res = pdsdp.solve_pd_sdp(prob, cfg)
            out[pre + f"X{K}"] = res.X.data
            out[pre + f"y{K}"] = res.y
            out[pre + f"res{K}"] = np.array(res.final_residuals)
        cfg = pdsdp.SolverConfig(eps_tol=1e-4, max_iter=3000, time_limit_s=1e9)
        res = pdsdp.solve_pd_sdp(prob, cfg)
        out[pre + "status"] = res.status.value
        out[pre + "iters"] = res.iterations
        out[pre + "X"] = res.X.data
        out[pre + "y"] = res.y
        out[pre + "pobj"] = res.primal_objective
        out[pre + "dobj"] = res.dual_objective
        out[pre + "res"] = np.array(res.final_residuals)
        out[pre + "scale"] = res.residual_scale
        print("pd", ci, prob.n, res.status, res.iterations, res.primal_objective)
    np.savez_compressed(path, **out)


def make_dense(path):
    """Reference outputs where its dense eigh path runs (symmat.py:158-161,
    181-185, 223-226) -- what the device's full eigensolver (dense_path.cuh)
    is checked against:
      * aproj_psd at n = 100 / 300 with 2 (r+1) > n or r + 1 above the eigen block;
      * exact PD-SDP (full projection each iteration) on an n = 100 Max-Cut;
      * an LR-PD-SDP run whose rank doubling crosses the eigen block limit
        with more positive eigenvalues than a block holds (equipartition n = 150)."""
    out = {}
    zs = np.random.default_rng(SKETCH_SEED).standard_normal((300, 4))
    for (n, seed, ranks) in ((100, 11, (60, 80, 100)), (300, 12, (100, 200, 300))):
        S = dense_case_matrix(n, seed)
        Sp = pdsdp.SymMatrix.from_dense(S)
        for r in ranks:
            P, lam = pdsdp.aproj_psd(Sp, r)
            pre = f"ap_n{n}_r{r}_"
            Pd = P.to_dense()
            out[pre + "lam"] = lam
            out[pre + "fro"] = np.linalg.norm(Pd)
            out[pre + "diag"] = np.diag(Pd).copy()
            out[pre + "Pz"] = Pd @ zs[:n]
            if n == 100:
                out[pre + "P"] = P.data
    prob = to_ref(workloads.maxcut_problem(100, 0.1, 0, signed=False))
    flatten_problem("pd_", prob, out)
    for K in (1, 10, 50):
        res = pdsdp.solve_pd_sdp(prob, pdsdp.SolverConfig(eps_tol=1e-4, max_iter=K, time_limit_s=1e9))
        out[f"pd_X{K}"] = res.X.data
        out[f"pd_y{K}"] = res.y
        out[f"pd_res{K}"] = np.array(res.final_residuals)
    res = pdsdp.solve_pd_sdp(prob, pdsdp.SolverConfig(eps_tol=1e-4, max_iter=5000, time_limit_s=1e9))
    out["pd_status"] = res.status.value
    out["pd_iters"] = res.iterations
    out["pd_X"] = res.X.data
    out["pd_y"] = res.y
    out["pd_pobj"] = res.primal_objective
    out["pd_dobj"] = res.dual_objective
    out["pd_res"] = np.array(res.final_residuals)
    print("dense pd", res.status, res.iterations, res.primal_objective)
    prob = to_ref(workloads.equipartition_problem(150, 0.05, 2))
    cfg = pdsdp.SolverConfig(eps_tol=1e-4, max_iter=300, initial_rank=70, window_ell=50, time_limit_s=1e9)
    with LambdaRecorder() as rec:
        res = pdsdp.solve_lr_pd_sdp(prob, cfg)
    out["lr_status"] = res.status.value
    out["lr_iters"] = res.iterations
    out["lr_X"] = res.X.data
    out["lr_y"] = res.y
    out["lr_res"] = np.array(res.final_residuals)
    out["lr_rank_path"] = np.array(res.rank_path)
    out["lr_lam"] = np.array(rec.values)
    out["lr_pobj"] = res.primal_objective
    w = np.linalg.eigvalsh(res.X.to_dense())
    out["lr_npos"] = int(np.sum(w > 1e-9 * w.max()))
    print("dense lr", res.status, res.iterations, res.rank_path, out["lr_npos"])
    # a Max-Cut whose first projection argument has ~n positive eigenvalues
    prob = to_ref(workloads.maxcut_problem(200, 0.1, 0, signed=False))
    res = pdsdp.solve_lr_pd_sdp(prob, pdsdp.SolverConfig(initial_rank=80, max_iter=2, time_limit_s=1e9))
    out["mc_X"] = res.X.data
    out["mc_y"] = res.y
    out["mc_res"] = np.array(res.final_residuals)
    np.savez_compressed(path, **out)


def make_mimo(path):
    """LR-PD-SDP on MIMO relaxations (reference instances.gen_mimo): n+1
    diagonal pins and the box -1 <= X_ij <= 1 as 2 n (n+1) / 2 inequality
    rows -- the inequality-heavy regime (proj_box branch of the dual step)."""
    out = {}
    for ci, (n, sigma, seed, K) in enumerate([(12, 0.3, 3, 400), (40, 0.5, 8, 60)]):
        prob = _mimo(n, sigma, seed)
        pre = f"c{ci}_"
        flatten_problem(pre, prob, out)
        cfg = pdsdp.SolverConfig(eps_tol=1e-4, max_iter=K, initial_rank=1, window_ell=50, time_limit_s=1e9)
        res = pdsdp.solve_lr_pd_sdp(prob, cfg)
        out[pre + "K"] = K
        out[pre + "status"] = res.status.value
        out[pre + "iters"] = res.iterations
        out[pre + "X"] = res.X.data
        out[pre + "y"] = res.y
        out[pre + "pobj"] = res.primal_objective
        out[pre + "dobj"] = res.dual_objective
        out[pre + "res"] = np.array(res.final_residuals)
        out[pre + "rank_path"] = np.array(res.rank_path)
        print("mimo", n, res.status, res.iterations, res.rank_path, res.primal_objective)
    np.savez_compressed(path, **out)


def make_check(path):
    """Reference problem.check_solution reports (objectives, violations,
    min eigenvalue, gap) on solver outputs and on perturbed / indefinite X."""
    from pdsdp.problem import check_solution
    rng = np.random.default_rng(99)
    out = {}
    cases = []
    d = np.load(os.path.join(HERE, "lr_small.npz"))
    for ci in (1, 2, 4):
        pre = f"c{ci}_"
        n = int(d[pre + "n"])
        cases.append((pre, n, d[pre + "X"], d[pre + "y"]))
    for k, (pre, n, Xd, y) in enumerate(cases):
        ref = RProblem
        indptr, idx, val = d[pre + "indptr"], d[pre + "idx"], d[pre + "val"]
        rows = [RRow(idx[indptr[i]:indptr[i + 1]], val[indptr[i]:indptr[i + 1]]) for i in range(len(indptr) - 1)]
        m = d[pre + "b"].size
        prob = ref(n=n, C=RSym(n, d[pre + "C"]), A=rows[:m], b=d[pre + "b"], G=rows[m:], h=d[pre + "h"])
        R = rng.standard_normal((n, n))
        Xs = [Xd, Xd + pdsdp.SymMatrix.from_dense(0.3 * (R + R.T)).data]
        for j, X in enumerate(Xs):
            rep = check_solution(prob, RSym(n, X.copy()), y)
            q = f"k{k}_{j}_"
            flatten_problem(q, prob, out)
            out[q + "X"] = X
            out[q + "yv"] = y
            out[q + "report"] = np.array([rep.primal_objective, rep.dual_objective, rep.equality_violation,
                                          rep.inequality_violation, rep.min_eigenvalue, rep.duality_gap])
    np.savez_compressed(path, **out)


SDPA_MULTIBLOCK = """* a two-block document: comments, braces, a diagonal block, a duplicate
"hand written"
3 =mdim
2 =nblocks
{3, -2}
{1.0, 2.5, -1.0}
0 1 1 1 2.0
0 1 1 3 -0.5
0 2 1 1 1.5
1 1 1 1 1.0
1 1 2 3 0.25
1 1 2 3 0.25
2 1 3 3 1.0
2 2 2 2 -2.0
3 1 1 2 1.0
3 2 1 1 4.0
"""

SDPA_BAD = [
    "1\n1\n2\n1.0\n0 1 2 1 1.0\n",            # lower triangle
    "1\n1\n2\n1.0\n0 1 1 3 1.0\n",            # outside the block
    "1\n1\n-2\n1.0\n0 1 1 2 1.0\n",           # off-diagonal in a diagonal block
    "1\n1\n2\n1.0\n0 1 1 1\n",                # 4 fields
    "1\n1\n2\nx\n0 1 1 1 1.0\n",              # non-numeric c
    "2\n1\n2\n1.0\n0 1 1 1 1.0\n",            # short c vector (takes an entry line)
    "1\n0\n2\n1.0\n0 1 1 1 1.0\n",            # zero blocks
    "1\n1\n2\n1.0\n3 1 1 1 1.0\n",            # matrix index out of range
    "1\n1\n2\n",                                  # too short
]


def make_io(path):
    """Reference io.py on SDPA / extended / solution documents."""
    from pdsdp import io as rio
    from pdsdp.problem import check_solution
    out = {}
    docs = {"cfg1": rio.write_sdpa(to_ref(workloads.config(0)[0])), "multi": SDPA_MULTIBLOCK}
    for name, text in docs.items():
        prob = rio.parse_sdpa(text)
        out[f"sdpa_{name}_text"] = np.array(text)
        flatten_problem(f"sdpa_{name}_", prob, out)
        out[f"sdpa_{name}_sign"] = prob.objective_sign
        out[f"sdpa_{name}_rewrite"] = np.array(rio.write_sdpa(prob))
    msgs = []
    for text in SDPA_BAD:
        try:
            rio.parse_sdpa(text)
            msgs.append("")
        except rio.ParseError as exc:
            msgs.append(str(exc))
    out["sdpa_bad_text"] = np.array(SDPA_BAD)
    out["sdpa_bad_msg"] = np.array(msgs)
    d = np.load(os.path.join(HERE, "lr_small.npz"))
    pre = "c1_"
    n = int(d[pre + "n"])
    indptr, idx, val = d[pre + "indptr"], d[pre + "idx"], d[pre + "val"]
    rows = [RRow(idx[indptr[i]:indptr[i + 1]], val[indptr[i]:indptr[i + 1]]) for i in range(len(indptr) - 1)]
    m = d[pre + "b"].size
    prob = RProblem(n=n, C=RSym(n, d[pre + "C"]), A=rows[:m], b=d[pre + "b"], G=rows[m:], h=d[pre + "h"],
                    name="lr_small_c1")
    ext = rio.write_extended(prob)
    out["ext_text"] = np.array(ext)
    p2 = rio.parse_extended(ext)
    flatten_problem("ext_", p2, out)
    cfg = pdsdp.SolverConfig(eps_tol=1e-4, max_iter=400, initial_rank=1, window_ell=50, time_limit_s=1e9)
    res = pdsdp.solve_lr_pd_sdp(prob, cfg)
    rep = check_solution(prob, res.X, res.y)
    out["sol_text"] = np.array(rio.write_solution(res, rep))
    np.savez_compressed(path, **out)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--big", action="store_true")
    ap.add_argument("--only", default="")
    ap.add_argument("--full", default="",
                    help="comma list of to-tolerance reference runs: cfg2, cfg4, cfg5sN (seed N), cfg1")
    a = ap.parse_args()
    if a.full:
        for name in a.full.split(","):
            if name == "cfg3_stall":
                # config 3 past its first stall-triggered rank doubling (k = 501):
                # pins the stall rule and the rank path at the full size
                make_sketch(os.path.join(HERE, "cfg3_stall_sketch.npz"), 2, (510,))
                continue
            if name.startswith("cfg5s"):
                make_full(os.path.join(HERE, f"{name}_full.npz"), 4, int(name[5:]))
            else:
                make_full(os.path.join(HERE, f"{name}_full.npz"), int(name[3:]) - 1)
        sys.exit(0)
    jobs = {
        "ops_small": lambda: make_ops_small(os.path.join(HERE, "ops_small.npz")),
        "lr_small": lambda: make_lr_small(os.path.join(HERE, "lr_small.npz")),
        "cfg1": lambda: make_cfg1(os.path.join(HERE, "cfg1.npz")),
        "pd_small": lambda: make_pd_small(os.path.join(HERE, "pd_small.npz")),
        "mimo": lambda: make_mimo(os.path.join(HERE, "mimo.npz")),
        "dense": lambda: make_dense(os.path.join(HERE, "dense.npz")),
        "check": lambda: make_check(os.path.join(HERE, "check.npz")),
        "io": lambda: make_io(os.path.join(HERE, "io.npz")),
    }
    if a.big:
        jobs["cfg2"] = lambda: make_sketch(os.path.join(HERE, "cfg2_sketch.npz"), 1, (1, 5))
        jobs["cfg4"] = lambda: make_sketch(os.path.join(HERE, "cfg4_sketch.npz"), 3, (1, 5))
        jobs["cfg5"] = lambda: make_sketch(os.path.join(HERE, "cfg5_sketch.npz"), 4, (1, 10))
        jobs["cfg3"] = lambda: make_sketch(os.path.join(HERE, "cfg3_sketch.npz"), 2, (1, 2))
    for name, fn in jobs.items():
        if a.only and name not in a.only.split(","):
            continue
        t = time.perf_counter()
        fn()
        print(name, f"{time.perf_counter() - t:.1f}s")
