"""Drop-in ``solve_lr_pd_sdp`` running the per-iteration hot path on a B200.

Host side of the boundary.  The control flow is the reference's Algorithm 2
driver (``pkg/src/pdsdp/lowrank.py:102-208``) statement for statement —
relative residual scale, checkpoints, rank certificate on lambda_{r+1}, stall
window, rank doubling, time limit, objectives — while every per-iteration
computation (``approximate_primal_step``, ``dual_step``, ``residuals``,
``_finite``) is one call into the sm_100a library, which returns scalars
only.  Iterates stay on the device; X and y are downloaded at checkpoints and
at the end (the reference copies them there too, ``lowrank.py:163-169``).
"""

from __future__ import annotations

import logging
import math
import time

import numpy as np

from .config import (
    DEFAULT_EPS_LAMBDA_PER_N,
    Checkpoint,
    ProgressCallback,
    ProgressInfo,
    RankController,
    SolveResult,
    SolveStatus,
    SolverConfig,
    rank_certificate_satisfied,
    stall_detected,
    update_rank,
)
from .device import (
    KMAX, OUT_EIGCONV, OUT_EPS_D, OUT_EPS_P, OUT_FINITE, OUT_LAMBDA, OUT_MATVECS, OUT_PASSES,
    DeviceBatch,
)
from .layout import SymMatrix, approx_error_bound
from .model import SdpProblem

logger = logging.getLogger(__name__)

# problem.py:21-26
_NORM_MIN_ITER = 200
_NORM_MAX_ITER = 10_000
_NORM_REL_TOL = 1e-10
_NORM_SAFETY = 1.0 + 1e-7
_NORM_CHUNK = 256
FLAG_COLD, FLAG_CERT, FLAG_RERUN = 1, 2, 4


def _device_batch(prob: SdpProblem) -> DeviceBatch:
    cache = prob._device_cache
    if "batch" not in cache:
        cache["batch"] = DeviceBatch([prob])
    return cache["batch"]


def operator_norm_on_device(batch: DeviceBatch, inst: int, seed: int = 0) -> float:
    """Seeded power iteration on M^T M (reference ``problem.py:157-185``).

    The start vectors come from the reference's own RNG stream on the host;
    each product runs on the device; the stopping rule is evaluated on the
    host over the device's per-iteration ||M x|| values, iteration by
    iteration, so the accepted estimate is the one the reference accepts."""
    prob = batch.problems[inst]
    P = prob.packed_len
    pos = batch.opnorm_positions(inst)
    if pos.size == 0:
        raise ValueError("all constraint rows are zero; operator norm is 0")
    rng = np.random.default_rng(seed)
    x = rng.standard_normal(P)
    x /= np.linalg.norm(x)
    start = x[pos]
    sigma = 0.0
    it = 0
    while it < _NORM_MAX_ITER:
        chunk = min(_NORM_CHUNK, _NORM_MAX_ITER - it)
        s_vals = batch.opnorm_run(inst, start, chunk)
        start = None
        advanced = chunk
        for j in range(chunk):
            s = float(s_vals[j])
            itj = it + j
            if s == 0.0:
                x = rng.standard_normal(P)
                x /= np.linalg.norm(x)
                start = x[pos]
                advanced = j + 1
                break
            if itj + 1 >= _NORM_MIN_ITER and abs(s - sigma) <= _NORM_REL_TOL * s:
                return s * _NORM_SAFETY
            sigma = s
        it += advanced
    return sigma * _NORM_SAFETY


def estimate_operator_norm(prob: SdpProblem, seed: int = 0) -> float:
    """Drop-in for ``problem.estimate_operator_norm`` (device products)."""
    return operator_norm_on_device(_device_batch(prob), 0, seed)


def step_size(prob: SdpProblem, config: SolverConfig) -> float:
    """reference ``pdhg.py:211-214``"""
    if config.alpha_override is not None:
        return config.alpha_override
    return config.alpha_safety / estimate_operator_norm(prob, config.seed)


class _DeviceIterate:
    """Device-resident (X_k, y_k) of one instance: which buffers hold what."""

    def __init__(self, batch: DeviceBatch, inst: int):
        self.batch, self.inst = batch, inst
        self.ypar = 0          # y_k is ybuf[ypar]
        self.which = 0         # X_k is the newest factor (0) or the previous one (1)
        self.k = 0

    def X(self) -> SymMatrix:
        n = self.batch.problems[self.inst].n
        if self.k == 0:
            return SymMatrix.zero(n)
        return SymMatrix(n, self.batch.download_x(self.inst, self.which))

    def y(self) -> np.ndarray:
        return self.batch.download_y(self.inst, self.ypar)

    def objective(self) -> float:
        if self.k == 0:
            return 0.0
        return self.batch.objective(self.inst, self.which)


class LoopOutcome:
    """What the host loop leaves behind (iterates stay on the device)."""

    def __init__(self, **kw):
        self.__dict__.update(kw)


def _stall_thresholds(controller: RankController, n: int, K: int) -> np.ndarray:
    """Smallest combined residual at which the stall rule (reference
    ``lowrank.py:64-69,181``) would fire at each of the next K steps: step j
    compares against the value ell steps back, already in the window when
    K <= ell; +inf where the rule cannot fire."""
    thr = np.full(K, np.inf)
    if controller.r >= n:
        return thr
    h = controller.history
    L, ell = len(h), controller.ell
    for j in range(K):
        if L + j + 1 >= ell + 1:
            thr[j] = h[L + j - ell]
    return thr


def run_lr_loop(batch: DeviceBatch, inst: int, prob: SdpProblem, config: SolverConfig,
                alpha: float, callback: ProgressCallback | None = None,
                t0: float | None = None, chunk: int = KMAX) -> LoopOutcome:
    """The ``for k`` loop of reference ``lowrank.py:125-190`` on a resident
    instance.  Iterations run on the device in chunks of up to ``chunk``; the
    device pauses at the first step where a convergence check, a stall or a
    divergence can fire, and the host then applies the reference's control
    logic to every executed step in order -- so every decision is taken at the
    same iteration, on the same scalars, as with one call per iteration."""
    t0 = time.perf_counter() if t0 is None else t0
    n = prob.n
    eps_lambda = (config.eps_lambda if config.eps_lambda is not None
                  else DEFAULT_EPS_LAMBDA_PER_N * n)
    controller = RankController(r=min(max(config.initial_rank, 1), n), ell=config.window_ell)
    batch.set_alpha(inst, alpha)
    batch.reset(inst, 0.0)
    it = _DeviceIterate(batch, inst)
    rank_path = [(0, controller.r)]
    status = None
    res = (math.nan, math.nan, math.nan)
    scale = 1.0
    eig_passes = eig_matvecs = eig_unconverged = 0
    k = 1
    while k <= config.max_iter and status is None:
        # chunk length: the first iteration alone (it fixes the relative
        # scale); never across a progress callback; at most window_ell
        K = 1 if k == 1 else min(chunk, config.max_iter - k + 1, controller.ell)
        if callback is not None:
            K = min(K, config.progress_every - (k - 1) % config.progress_every)
        conv = config.eps_tol * scale if k > 1 else -1.0
        stall = _stall_thresholds(controller, n, K)
        outs, done = batch.iterate_many([inst], [controller.r], [it.ypar], K, [conv], stall)
        outs, done = outs[0], int(done[0])
        for j in range(done):
            out = outs[j]
            eig_passes += int(out[OUT_PASSES])
            eig_matvecs += int(out[OUT_MATVECS])
            if out[OUT_FINITE] == 1.0:
                ec = float(out[OUT_EPS_P]) + float(out[OUT_EPS_D])
                sc = (1.0 + ec) if (k == 1 and config.relative_residuals) else scale
                if ec <= config.eps_tol * sc:
                    # checkpoint iteration: the certificate needs lambda_{r+1} to the
                    # reference's accuracy; re-run this iteration from the same
                    # (X_k, y_k) with the certificate eigenpair converged too
                    assert j == done - 1, "device chunk ran past a checkpoint"
                    out = batch.iterate([inst], [controller.r], [it.ypar], [FLAG_CERT | FLAG_RERUN])[0]
                    eig_passes += int(out[OUT_PASSES])
                    eig_matvecs += int(out[OUT_MATVECS])
            if out[OUT_EIGCONV] == 0:
                eig_unconverged += 1
                logger.info("eigensolver hit its pass limit at k=%d (r=%d)", k, controller.r)
            if out[OUT_FINITE] != 1.0:                   # _finite, lowrank.py:145-147
                status = SolveStatus.DIVERGED
                it.which = 1
                break
            it.k = k                                     # state.advance, pdhg.py:113-118
            it.ypar ^= 1
            it.which = 0
            lambda_r = float(out[OUT_LAMBDA])
            controller.last_lambda_r = lambda_r
            ep, ed = float(out[OUT_EPS_P]), float(out[OUT_EPS_D])
            res = (ep, ed, ep + ed)
            controller.history.append(res[2])
            if k == 1 and config.relative_residuals:
                scale = 1.0 + res[2]
            if callback is not None and k % config.progress_every == 0:
                callback(ProgressInfo(k, *res, controller.r, it.objective()))
            if res[2] <= config.eps_tol * scale:
                Xc = it.X()
                controller.checkpoints.append(
                    Checkpoint(controller.r, Xc, it.y(), prob.C.inner(Xc)))
                if rank_certificate_satisfied(n, controller.r, lambda_r, eps_lambda):
                    status = SolveStatus.OPTIMAL
                    break
                logger.debug("converged at rank %d but certificate %.3e > %.3e; doubling",
                             controller.r, approx_error_bound(n, controller.r, lambda_r), eps_lambda)
                update_rank(controller, n)
                rank_path.append((k, controller.r))
                assert j == done - 1, "device chunk ran past a rank change"
            elif controller.r < n and stall_detected(controller.history, controller.ell):
                logger.debug("stalled at rank %d after %d iterations; doubling", controller.r, k)
                update_rank(controller, n)
                rank_path.append((k, controller.r))
                assert j == done - 1, "device chunk ran past a stall"
            k += 1
        # time limit: checked at chunk granularity (the device pauses only at
        # algorithmic events)
        if status is None and time.perf_counter() - t0 > config.time_limit_s:
            status = SolveStatus.TIME_LIMIT
    if status is None:
        status = SolveStatus.MAX_ITERATIONS
    return LoopOutcome(status=status, it=it, res=res, rank_path=rank_path, controller=controller,
                       scale=scale, eig_passes=eig_passes, eig_matvecs=eig_matvecs,
                       eig_unconverged=eig_unconverged)


def solve_lr_pd_sdp(
    prob: SdpProblem,
    config: SolverConfig | None = None,
    callback: ProgressCallback | None = None,
    *,
    stats: dict | None = None,
) -> SolveResult:
    """Rank-adaptive primal-dual iteration from a zero start
    (reference ``lowrank.py:102-208``); per-iteration work on the B200."""
    config = config or SolverConfig()
    config.validate()
    t0 = time.perf_counter()
    batch = _device_batch(prob)
    alpha = step_size(prob, config)
    o = run_lr_loop(batch, 0, prob, config, alpha, callback, t0)
    X = o.it.X()
    y = o.it.y()
    pobj = prob.C.inner(X)                               # lowrank.py:191-194
    dobj = -float(prob.b @ y[: prob.m] + prob.h @ y[prob.m:])
    if stats is not None:
        stats.update(eig_passes=o.eig_passes, eig_matvecs=o.eig_matvecs,
                     eig_unconverged=o.eig_unconverged, alpha=alpha)
    return SolveResult(
        status=o.status, X=X, y=y, primal_objective=pobj, dual_objective=dobj,
        final_residuals=o.res, iterations=o.it.k, rank_path=o.rank_path,
        checkpoints=o.controller.checkpoints, wall_time_s=time.perf_counter() - t0,
        residual_scale=o.scale, objective_sign=prob.objective_sign,
    )
