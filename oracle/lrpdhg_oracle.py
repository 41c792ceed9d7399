"""CPU ORACLE — test infrastructure only, never the product path.

A numpy/scipy restatement of the reference's LR-PD-SDP hot path
(``/root/reference/pkg/src/pdsdp``; Algorithm 2 of arXiv 1810.05231).  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` leg may import it, and only as the checker or the timed
CPU baseline.  The product (``paper_1810_05231_b200``) never imports this
module; it fails loudly when its CUDA library is missing.

The arithmetic the reference delegates to third-party code is delegated to the
same third-party code here: numpy 2.3 LAPACK ``eigh`` (``symmat.py:158-161``),
scipy 1.18 ARPACK ``eigsh`` (``symmat.py:189-199``) and scipy.sparse CSR
products (``problem.py:140-154``).  The pinned versions are those installed in
this image (the reference declares only ``numpy>=1.24``, ``scipy>=1.10``,
``pyproject.toml:10-13``).

Pinning: ``tests/golden/make_golden.py`` runs the reference itself (in the
build container, where ``/root/reference`` exists) and stores its outputs;
``tests/test_oracle_golden.py`` checks this restatement against them and
against the known-answer cases of the reference's own unit tests.

One deliberate deviation, documented in SURVEY.md §8c quirk (1): when ARPACK
raises ``ArpackError`` (e.g. "starting vector is zero" when S + cI vanishes,
BASELINE config 4 iteration 1) the reference crashes; the oracle takes the
same dense fallback the reference takes for ``ArpackNoConvergence``
(``symmat.py:200-207``).
"""

from __future__ import annotations

import math
import time
from collections import deque

import numpy as np
import scipy.sparse as sp
from scipy.sparse.linalg import ArpackError, ArpackNoConvergence, eigsh

R2 = math.sqrt(2.0)

# symmat.py:31-34
KRYLOV_SEED = 0x5EED
KRYLOV_MAXITER = 300
KRYLOV_TOL = 1e-12
DENSE_DIM = 32
# problem.py:21-26
NORM_MIN_IT, NORM_MAX_IT, NORM_RTOL, NORM_SAFETY = 200, 10_000, 1e-10, 1.0 + 1e-7


# ----------------------------------------------------------------------------
# packed layout (symmat.py:50-101)

def tri(n):
    return np.triu_indices(n)


def pack(S):
    """symmat.py:66-86 (symmetrise, scale off-diagonals by sqrt 2)."""
    n = S.shape[0]
    iu, ju = tri(n)
    v = 0.5 * (S[iu, ju] + S[ju, iu])
    v[iu != ju] *= R2
    return v


def unpack(v, n):
    """symmat.py:89-101."""
    iu, ju = tri(n)
    w = v.copy()
    w[iu != ju] /= R2
    S = np.zeros((n, n))
    S[iu, ju] = w
    S[ju, iu] = w
    return S


# ----------------------------------------------------------------------------
# eigen-decompositions and projections (symmat.py:158-245)

def eig_desc(S_dense):
    """symmat.py:158-161: all pairs, descending."""
    w, V = np.linalg.eigh(S_dense)
    return w[::-1].copy(), V[:, ::-1].copy()


def top_eigen(Sp, n, k):
    """symmat.py:170-209: k largest-algebraic pairs of the packed matrix."""
    if not 1 <= k <= n:
        raise ValueError(f"rank r={k} outside [1, {n}]")
    dense = unpack(Sp, n)
    if n <= DENSE_DIM or 2 * k > n:
        w, V = eig_desc(dense)
        return w[:k].copy(), V[:, :k].copy(), "dense"
    c = float(np.abs(dense).sum(axis=1).max())
    dense[np.diag_indices(n)] += c
    v0 = np.random.default_rng(KRYLOV_SEED).standard_normal(n)
    v0 /= np.linalg.norm(v0)
    try:
        w, V = eigsh(dense, k=k, which="LA", v0=v0, ncv=min(n, max(2 * k + 1, 20)),
                     maxiter=KRYLOV_MAXITER, tol=KRYLOV_TOL)
    except (ArpackNoConvergence, ArpackError):
        w, V = eig_desc(unpack(Sp, n))
        return w[:k].copy(), V[:, :k].copy(), "fallback"
    o = np.argsort(w)[::-1]
    return w[o] - c, V[:, o], "arpack"


def clip_assemble(w, V, n):
    """symmat.py:212-220: sum of max(lambda,0) u u^T, packed."""
    keep = w > 0.0
    if not np.any(keep):
        return np.zeros(n * (n + 1) // 2)
    U = V[:, keep]
    P = (U * w[keep]) @ U.T
    return pack(0.5 * (P + P.T))


def proj_psd(Sp, n):
    """symmat.py:223-226."""
    w, V = eig_desc(unpack(Sp, n))
    return clip_assemble(w, V, n)


def aproj_psd(Sp, n, r):
    """symmat.py:229-245: rank-r projection and the certificate eigenvalue
    lambda_{min(r+1, n)}."""
    if not 1 <= r <= n:
        raise ValueError(f"rank r={r} outside [1, {n}]")
    k = min(r + 1, n)
    w, V, _ = top_eigen(Sp, n, k)
    return clip_assemble(w[:r], V[:, :r], n), float(w[k - 1])


# ----------------------------------------------------------------------------
# linear maps (problem.py:119-185)

def stacked_csr(prob):
    indptr, idx, val = prob.stacked_arrays()
    return sp.csr_matrix((val, idx, indptr), shape=(prob.m + prob.p, prob.packed_len))


def op_norm(M, seed=0):
    """problem.py:157-185: power iteration on M^T M, seeded start."""
    rng = np.random.default_rng(seed)
    P = M.shape[1]
    x = rng.standard_normal(P)
    x /= np.linalg.norm(x)
    sigma = 0.0
    for it in range(NORM_MAX_IT):
        y = M @ x
        s = float(np.linalg.norm(y))
        if s == 0.0:
            x = rng.standard_normal(P)
            x /= np.linalg.norm(x)
            continue
        x = M.T @ y
        x /= np.linalg.norm(x)
        if it + 1 >= NORM_MIN_IT and abs(s - sigma) <= NORM_RTOL * s:
            sigma = s
            break
        sigma = s
    return sigma * NORM_SAFETY


def box_resolvent(u, alpha, b, h):
    """pdhg.py:143-163: u - alpha * [b; min(u2/alpha, h)]."""
    m = b.size
    t = u / alpha
    proj = np.empty_like(u)
    proj[:m] = b
    proj[m:] = np.minimum(t[m:], h)
    return u - alpha * proj


def dual_update(M, y, Xn, Xo, alpha, b, h):
    """pdhg.py:185-195."""
    return box_resolvent(y + alpha * (M @ (2.0 * Xn - Xo)), alpha, b, h)


def fixed_point_residuals(M, Xn, Xo, yn, yo, alpha):
    """pdhg.py:198-208."""
    dX = Xn - Xo
    dy = yn - yo
    ep = float(np.linalg.norm(dX / alpha - M.T @ dy))
    ed = float(np.linalg.norm(dy / alpha - M @ dX))
    return ep, ed, ep + ed


# ----------------------------------------------------------------------------
# Algorithm 2 driver (lowrank.py:102-208)

class OracleResult(dict):
    __getattr__ = dict.__getitem__


def solve_lr(prob, cfg, record_at=(), progress=None, alpha=None, stop_after=None):
    """Run Algorithm 2 exactly as ``lowrank.solve_lr_pd_sdp`` does.

    Returns a dict with status, X (packed), y, objectives, residuals,
    iterations, rank_path, checkpoints [(rank, obj)], residual_scale, plus
    ``snapshots``: {k: (X packed, y, lambda_{r+1}, residuals)} for k in
    ``record_at`` and ``history``: per-iteration (eps_p, eps_d, eps_c, r).
    ``stop_after`` truncates the run after that many iterations (CPU
    baseline sampling); ``alpha`` skips the operator-norm estimate.
    """
    cfg.validate()
    t0 = time.perf_counter()
    n = prob.n
    M = stacked_csr(prob)
    C = prob.C.data
    if alpha is None:
        alpha = cfg.alpha_override if cfg.alpha_override is not None else \
            cfg.alpha_safety / op_norm(M, cfg.seed)
    eps_lambda = cfg.eps_lambda if cfg.eps_lambda is not None else 5e-2 * n
    r = min(max(cfg.initial_rank, 1), n)
    window = deque(maxlen=cfg.window_ell + 1)
    X = np.zeros(n * (n + 1) // 2)
    y = np.zeros(prob.m + prob.p)
    rank_path = [(0, r)]
    checkpoints = []
    snaps, hist = {}, []
    record_at = set(record_at)
    status = None
    res = (math.nan, math.nan, math.nan)
    scale = 1.0
    k_done = 0
    for k in range(1, cfg.max_iter + 1):
        S = X - alpha * (M.T @ y + C)                      # lowrank.py:97-98
        Xn, lam = aproj_psd(S, n, r)                       # symmat.py:229-245
        yn = dual_update(M, y, Xn, X, alpha, prob.b, prob.h)
        if not (np.all(np.isfinite(Xn)) and np.all(np.isfinite(yn))):
            status = "diverged"
            break
        res = fixed_point_residuals(M, Xn, X, yn, y, alpha)
        X, y = Xn, yn
        k_done = k
        window.append(res[2])
        hist.append((*res, r))
        if k in record_at:
            snaps[k] = (X.copy(), y.copy(), lam, res)
        if k == 1 and cfg.relative_residuals:
            scale = 1.0 + res[2]
        if progress is not None and k % cfg.progress_every == 0:
            progress((k, *res, r, float(C @ X)))
        if res[2] <= cfg.eps_tol * scale:
            checkpoints.append((r, float(C @ X)))
            if (n - r) * max(lam, 0.0) <= eps_lambda:
                status = "optimal"
                break
            r = min(2 * r, n)
            window.clear()
            rank_path.append((k, r))
        elif r < n and len(window) >= cfg.window_ell + 1 and window[-1] >= window[-1 - cfg.window_ell]:
            r = min(2 * r, n)
            window.clear()
            rank_path.append((k, r))
        if time.perf_counter() - t0 > cfg.time_limit_s:
            status = "time_limit"
            break
        if stop_after is not None and k >= stop_after:
            status = "sampled"
            break
    if status is None:
        status = "max_iterations"
    return OracleResult(
        status=status, X=X, y=y, alpha=alpha,
        primal_objective=float(C @ X),
        dual_objective=-float(prob.b @ y[:prob.m] + prob.h @ y[prob.m:]),
        final_residuals=res, iterations=k_done, rank_path=rank_path,
        checkpoints=checkpoints, residual_scale=scale, snapshots=snaps,
        history=hist, wall_time_s=time.perf_counter() - t0,
    )


# ----------------------------------------------------------------------------
# Exact PD-SDP driver (pdhg.py:221-288) and the solution report
# (problem.py:213-240) -- checkers for SURVEY.md 8(f) rows 1 and 2.

def solve_pd(prob, cfg, alpha=None):
    """``pdhg.solve_pd_sdp``: X+ = proj_psd(X - alpha (M^T y + C)) with the
    full eigendecomposition, the same dual step and residuals, relative stop."""
    cfg.validate()
    t0 = time.perf_counter()
    n = prob.n
    M = stacked_csr(prob)
    C = prob.C.data
    if alpha is None:
        alpha = cfg.alpha_override if cfg.alpha_override is not None else \
            cfg.alpha_safety / op_norm(M, cfg.seed)
    X = np.zeros(n * (n + 1) // 2)
    y = np.zeros(prob.m + prob.p)
    status, res, scale, k_done = None, (math.nan,) * 3, 1.0, 0
    for k in range(1, cfg.max_iter + 1):
        Xn = proj_psd(X - alpha * (M.T @ y + C), n)           # pdhg.py:166-174
        yn = dual_update(M, y, Xn, X, alpha, prob.b, prob.h)
        if not (np.all(np.isfinite(Xn)) and np.all(np.isfinite(yn))):
            status = "diverged"
            break
        res = fixed_point_residuals(M, Xn, X, yn, y, alpha)
        X, y, k_done = Xn, yn, k
        if k == 1 and cfg.relative_residuals:
            scale = 1.0 + res[2]
        if res[2] <= cfg.eps_tol * scale:
            status = "optimal"
            break
        if time.perf_counter() - t0 > cfg.time_limit_s:
            status = "time_limit"
            break
    if status is None:
        status = "max_iterations"
    return OracleResult(status=status, X=X, y=y, iterations=k_done, final_residuals=res,
                        primal_objective=float(C @ X),
                        dual_objective=-float(prob.b @ y[:prob.m] + prob.h @ y[prob.m:]),
                        residual_scale=scale)


def check_solution(prob, Xp, y):
    """``problem.check_solution``: (pobj, dobj, eq. violation, ineq.
    violation, min eigenvalue, gap)."""
    M = stacked_csr(prob)
    mx = M @ Xp
    eq = float(np.linalg.norm(mx[:prob.m] - prob.b))
    ineq = float(np.linalg.norm(np.maximum(mx[prob.m:] - prob.h, 0.0)))
    pobj = float(prob.C.data @ Xp)
    dobj = -float(prob.b @ y[:prob.m] + prob.h @ y[prob.m:])
    lmin = float(np.linalg.eigvalsh(unpack(Xp, prob.n)).min())
    return np.array([pobj, dobj, eq, ineq, lmin, pobj - dobj])
