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
    SolutionReport,
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
    BLOCK_MAX, KMAX, OUT_EIGCONV, OUT_EPS_D, OUT_EPS_P, OUT_ERR, OUT_FINITE, OUT_LAMBDA, OUT_MATVECS,
    OUT_PASSES, DeviceBatch,
)
from .layout import SymMatrix, approx_error_bound
from .model import SdpProblem, as_problem

logger = logging.getLogger(__name__)

# problem.py:21-26
_NORM_MIN_ITER = 200
_NORM_MAX_ITER = 10_000
_NORM_REL_TOL = 1e-10
_NORM_SAFETY = 1.0 + 1e-7
_NORM_CHUNK = 256
FLAG_COLD, FLAG_CERT, FLAG_RERUN = 1, 2, 4
# Extra guard columns of the eigen block (flags bits 8..11).  One guard is
# fastest when an iteration converges in one or two filter passes (configs 2
# and 5); instances whose iterations keep needing many passes (config 4: a
# kept eigenvalue inside a cluster at a 1e-3 gap ratio) get a wider block:
# +2 columns at a rank change (where the block is rebuilt anyway) if the rank
# phase that just ended averaged more than GUARD_PASSES passes per iteration,
# up to GUARD_MAX.
GUARD_SHIFT, GUARD_STEP, GUARD_MAX, GUARD_PASSES = 8, 2, 6, 3.0


def _device_batch(prob: SdpProblem) -> DeviceBatch:
    """The resident single-instance batch of ``prob`` (created on first use);
    reference-typed problems go through :func:`~.model.as_problem`."""
    prob = as_problem(prob)
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


class _InstanceRun:
    """Host-side Algorithm-2 state of one instance (reference lowrank.py:115-190)."""

    def __init__(self, batch: DeviceBatch, inst: int, prob: SdpProblem, config: SolverConfig,
                 alpha: float, callback: ProgressCallback | None, t0: float):
        self.batch, self.inst, self.prob, self.config = batch, inst, prob, config
        self.callback, self.t0 = callback, t0
        n = prob.n
        self.n = n
        self.eps_lambda = (config.eps_lambda if config.eps_lambda is not None
                           else DEFAULT_EPS_LAMBDA_PER_N * n)
        self.controller = RankController(r=min(max(config.initial_rank, 1), n), ell=config.window_ell)
        batch.set_alpha(inst, alpha)
        batch.reset(inst, 0.0)
        self.it = _DeviceIterate(batch, inst)
        self.rank_path = [(0, self.controller.r)]
        self.status = None
        self.res = (math.nan, math.nan, math.nan)
        self.scale = 1.0
        self.k = 1
        self.eig_passes = self.eig_matvecs = self.eig_unconverged = 0
        self.dense = False     # dense-iterate mode (full device eigendecomposition)
        self.dense_from = None
        self.guard = 0         # extra guard columns of the eigen block
        self.phase_passes, self.phase_steps = 0.0, 0

    def flags(self) -> int:
        return self.guard << GUARD_SHIFT

    def _adapt_guard(self, outs, done: int) -> None:
        """Filter passes of the current rank phase (for the guard policy)."""
        if done > 0:
            self.phase_passes += float(np.asarray(outs[:done])[:, OUT_PASSES].sum())
            self.phase_steps += done

    def _rank_changed(self) -> None:
        if self.phase_steps >= 8 and self.phase_passes > GUARD_PASSES * self.phase_steps:
            self.guard = min(GUARD_MAX, self.guard + GUARD_STEP)
        self.phase_passes, self.phase_steps = 0.0, 0

    def enter_dense(self) -> None:
        """The projection argument has more positive eigenvalues than an eigen
        block holds (the unfinished step left X_k, y_k intact): continue with
        the full eigendecomposition, as the reference's dense fallback does
        (``symmat.py:181-185``)."""
        logger.info("k=%d (r=%d): eigen block limit reached, continuing with the dense device eigensolver",
                    self.k, self.controller.r)
        self.batch.dense_begin(self.inst, True)
        self.dense = True
        self.dense_from = self.k

    def step(self, chunk: int) -> None:
        """Run the next chunk of iterations of this instance alone."""
        if self.dense:
            out = self.batch.iterate_dense(self.inst, self.controller.r, self.it.ypar)
            self.consume([out], 1)
        else:
            K = self.max_chunk(chunk)
            conv, stall = self.thresholds(K)
            outs, done = self.batch.iterate_many([self.inst], [self.controller.r], [self.it.ypar], K, [conv], stall,
                                                 flags=[self.flags()])
            self.after_chunk(outs[0], int(done[0]), K)
        self.check_time()

    def after_chunk(self, outs, done: int, K: int) -> None:
        self._adapt_guard(outs, done)
        self.consume(outs, done)
        if self.status is None and done < K and outs[done][OUT_ERR] != 0.0:
            self.enter_dense()

    def max_chunk(self, chunk: int) -> int:
        """Steps the device may run before the host must look: the first
        iteration alone (it fixes the relative scale), never past max_iter, a
        progress callback, or window_ell steps (the stall thresholds must be
        known in advance)."""
        c = self.config
        if self.k == 1:
            return 1
        K = min(chunk, c.max_iter - self.k + 1, self.controller.ell)
        if self.callback is not None:
            K = min(K, c.progress_every - (self.k - 1) % c.progress_every)
        return max(K, 1)

    def thresholds(self, K: int):
        conv = self.config.eps_tol * self.scale if self.k > 1 else -1.0
        return conv, _stall_thresholds(self.controller, self.n, K)

    def consume(self, outs, done: int) -> None:
        """Apply the reference's per-iteration control logic to the executed
        steps, in order (lowrank.py:141-188).  The device pauses a chunk at the
        first step where that logic can act, so every step but the last is
        uneventful (finite, above the convergence threshold, below its stall
        threshold, no callback due): those are folded in at once after
        checking exactly that; anything else takes the step-by-step path."""
        nb = done - 1
        if nb >= 1 and self.k > 1 and self._bulk_ok(outs, nb):
            o = np.asarray(outs[:nb])
            self.eig_passes += int(o[:, OUT_PASSES].sum())
            self.eig_matvecs += int(o[:, OUT_MATVECS].sum())
            self.eig_unconverged += int(np.count_nonzero(o[:, OUT_EIGCONV] == 0))
            ep, ed = o[:, OUT_EPS_P], o[:, OUT_EPS_D]
            ec = ep + ed
            it, ctl = self.it, self.controller
            it.k = self.k + nb - 1
            it.ypar ^= nb & 1
            it.which = 0
            ctl.last_lambda_r = float(o[nb - 1, OUT_LAMBDA])
            self.res = (float(ep[-1]), float(ed[-1]), float(ec[-1]))
            ctl.history.extend(ec.tolist())
            self.k += nb
            self._consume_steps(outs, nb, done)
        else:
            self._consume_steps(outs, 0, done)

    def _bulk_ok(self, outs, nb: int) -> bool:
        c, ctl = self.config, self.controller
        o = np.asarray(outs[:nb])
        if not np.all(o[:, OUT_FINITE] == 1.0):
            return False
        ec = o[:, OUT_EPS_P] + o[:, OUT_EPS_D]
        if np.any(ec <= c.eps_tol * self.scale):
            return False
        if np.any(ec >= _stall_thresholds(ctl, self.n, nb)):
            return False
        if self.callback is not None:
            ks = self.k + np.arange(nb)
            if np.any(ks % c.progress_every == 0):
                return False
        return True

    def _consume_steps(self, outs, j0: int, done: int) -> None:
        c, ctl, it, n = self.config, self.controller, self.it, self.n
        for j in range(j0, done):
            out = outs[j]
            self.eig_passes += int(out[OUT_PASSES])
            self.eig_matvecs += int(out[OUT_MATVECS])
            if out[OUT_FINITE] == 1.0:
                ec = float(out[OUT_EPS_P]) + float(out[OUT_EPS_D])
                sc = (1.0 + ec) if (self.k == 1 and c.relative_residuals) else self.scale
                if ec <= c.eps_tol * sc and not self.dense:
                    # checkpoint iteration: the certificate needs lambda_{r+1} to the
                    # reference's accuracy; re-run this iteration from the same
                    # (X_k, y_k) with the certificate eigenpair converged too
                    assert j == done - 1, "device chunk ran past a checkpoint"
                    out = self.batch.iterate([self.inst], [ctl.r], [it.ypar], [FLAG_CERT | FLAG_RERUN | self.flags()])[0]
                    if out[OUT_ERR] != 0.0:
                        raise RuntimeError("certificate re-run exceeded the eigen block limit")
                    self.eig_passes += int(out[OUT_PASSES])
                    self.eig_matvecs += int(out[OUT_MATVECS])
            if out[OUT_EIGCONV] == 0:
                self.eig_unconverged += 1
                logger.info("eigensolver hit its pass limit at k=%d (r=%d)", self.k, ctl.r)
            if out[OUT_FINITE] != 1.0:                   # _finite, lowrank.py:145-147
                self.status = SolveStatus.DIVERGED
                it.which = 1
                return
            it.k = self.k                                # state.advance, pdhg.py:113-118
            it.ypar ^= 1
            it.which = 0
            lambda_r = float(out[OUT_LAMBDA])
            ctl.last_lambda_r = lambda_r
            ep, ed = float(out[OUT_EPS_P]), float(out[OUT_EPS_D])
            self.res = (ep, ed, ep + ed)
            ctl.history.append(self.res[2])
            if self.k == 1 and c.relative_residuals:
                self.scale = 1.0 + self.res[2]
            if self.callback is not None and self.k % c.progress_every == 0:
                self.callback(ProgressInfo(self.k, *self.res, ctl.r, it.objective()))
            k = self.k
            self.k += 1
            if self.res[2] <= c.eps_tol * self.scale:
                Xc = it.X()
                ctl.checkpoints.append(Checkpoint(ctl.r, Xc, it.y(), self.prob.C.inner(Xc)))
                if rank_certificate_satisfied(n, ctl.r, lambda_r, self.eps_lambda):
                    self.status = SolveStatus.OPTIMAL
                    return
                logger.debug("converged at rank %d but certificate %.3e > %.3e; doubling",
                             ctl.r, approx_error_bound(n, ctl.r, lambda_r), self.eps_lambda)
                update_rank(ctl, n)
                self.rank_path.append((k, ctl.r))
                self._rank_changed()
                assert j == done - 1, "device chunk ran past a rank change"
            elif ctl.r < n and stall_detected(ctl.history, ctl.ell):
                logger.debug("stalled at rank %d after %d iterations; doubling", ctl.r, k)
                update_rank(ctl, n)
                self.rank_path.append((k, ctl.r))
                self._rank_changed()
                assert j == done - 1, "device chunk ran past a stall"

    def check_time(self) -> None:
        # time limit at chunk granularity (the device pauses only at algorithmic events)
        if self.status is None and time.perf_counter() - self.t0 > self.config.time_limit_s:
            self.status = SolveStatus.TIME_LIMIT
        if self.status is None and self.k > self.config.max_iter:
            self.status = SolveStatus.MAX_ITERATIONS

    def outcome(self) -> LoopOutcome:
        return LoopOutcome(status=self.status or SolveStatus.MAX_ITERATIONS, it=self.it, res=self.res,
                           rank_path=self.rank_path, controller=self.controller, scale=self.scale,
                           eig_passes=self.eig_passes, eig_matvecs=self.eig_matvecs,
                           eig_unconverged=self.eig_unconverged)


def run_lr_loop(batch: DeviceBatch, inst: int, prob: SdpProblem, config: SolverConfig,
                alpha: float, callback: ProgressCallback | None = None,
                t0: float | None = None, chunk: int = KMAX) -> LoopOutcome:
    """The ``for k`` loop of reference ``lowrank.py:125-190`` on a resident
    instance.  Iterations run on the device in chunks of up to ``chunk``; the
    device pauses at the first step where a convergence check, a stall or a
    divergence can fire, and the host then applies the reference's control
    logic to every executed step in order -- so every decision is taken at the
    same iteration, on the same scalars, as with one call per iteration."""
    run = _InstanceRun(batch, inst, prob, config, alpha, callback,
                       time.perf_counter() if t0 is None else t0)
    while run.status is None:
        run.step(chunk)
    return run.outcome()


def run_lr_batch(batch: DeviceBatch, insts, config: SolverConfig, alphas,
                 chunk: int = KMAX, t0: float | None = None) -> list:
    """Algorithm 2 on many resident instances at once (the multi-instance
    analogue of the reference's sequential bench rows, ``cli.py:284-329``).

    Device-side scheduling: as many per-instance chunks as clusters of the
    iteration kernel fit on the GPU run side by side, one stream ("slot")
    each.  A chunk pauses on the device at its instance's own events; the host
    polls the slots, applies that instance's control logic (exactly as
    run_lr_loop does) and hands the freed slot to the next waiting instance, so
    no instance waits for another one's chunk and the batch takes about as long
    as its longest solve."""
    from collections import deque
    t0 = time.perf_counter() if t0 is None else t0
    runs = [_InstanceRun(batch, i, batch.problems[i], config, a, None, t0) for i, a in zip(insts, alphas)]
    nslots = batch.slots()
    free = list(range(nslots))
    inflight = {}
    queue = deque(runs)
    while queue or inflight:
        while free and queue:
            r = queue.popleft()
            if r.status is not None:
                continue
            if r.dense:                    # dense-path instances step alone, synchronously
                r.step(chunk)
                if r.status is None:
                    queue.append(r)
                continue
            K = r.max_chunk(chunk)
            conv, stall = r.thresholds(K)
            slot = free.pop()
            batch.chunk_launch(slot, r.inst, r.controller.r, r.it.ypar, K, conv, stall, flags=r.flags())
            inflight[slot] = (r, K)
        progressed = False
        for slot in list(inflight):
            if batch.chunk_poll(slot):
                r, K = inflight.pop(slot)
                outs, done = batch.chunk_collect(slot, r.inst, K)
                r.after_chunk(outs, done, K)
                r.check_time()
                free.append(slot)
                if r.status is None:
                    queue.append(r)
                progressed = True
        if not progressed and inflight:
            time.sleep(0)
    return [r.outcome() for r in runs]


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
    prob = as_problem(prob)
    batch = _device_batch(prob)
    alpha = step_size(prob, config)
    o = run_lr_loop(batch, 0, prob, config, alpha, callback, t0)
    return _result(prob, config, o, alpha, t0, stats)


def _result(prob, config, o, alpha, t0, stats=None) -> SolveResult:
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


def solve_lr_pd_sdp_batch(problems, config: SolverConfig | None = None) -> list:
    """Independent instances solved together on this GPU (BASELINE config 5):
    one resident batch, one cluster per instance per iteration, host control
    per instance.  Returns one SolveResult per problem, as solve_lr_pd_sdp."""
    config = config or SolverConfig()
    config.validate()
    t0 = time.perf_counter()
    problems = [as_problem(p) for p in problems]
    batch = DeviceBatch(problems)
    alphas = [config.alpha_override if config.alpha_override is not None else
              config.alpha_safety / operator_norm_on_device(batch, i, config.seed)
              for i in range(batch.count)]
    outs = run_lr_batch(batch, list(range(batch.count)), config, alphas, t0=t0)
    results = [_result(p, config, o, a, t0) for p, o, a in zip(problems, outs, alphas)]
    batch.close()
    return results


# ---------------------------------------------------------------------------
# Exact PD-SDP (reference pdhg.py:221-288) with the full PSD projection
# (symmat.py:223-226).  For n <= PDSDP_BLOCK_MAX the full projection is the
# eigen block covering all of R^n (r = n: the Rayleigh-Ritz step is then the
# complete eigendecomposition, one cluster kernel per iteration); larger n run
# on the dense-iterate path (csrc/dense_path.cuh: dense X_k in HBM, full
# one-sided-Jacobi eigendecomposition per iteration).


def solve_pd_sdp(
    prob: SdpProblem,
    config: SolverConfig | None = None,
    callback: ProgressCallback | None = None,
) -> SolveResult:
    """Exact primal-dual iteration from a zero start (reference
    ``pdhg.py:221-288``): X+ = proj_psd(X - alpha (M^T y + C)), the dual step
    and residuals as in the LR solver, stop on the (relative) combined
    residual, no rank control (``rank_path = [(0, n)]``)."""
    config = config or SolverConfig()
    config.validate()
    prob = as_problem(prob)
    n = prob.n
    t0 = time.perf_counter()
    alpha = step_size(prob, config)
    batch = _device_batch(prob)
    batch.set_alpha(0, alpha)
    batch.reset(0, 0.0)
    dense = n > BLOCK_MAX
    if dense:
        batch.dense_begin(0, False)
    it = _DeviceIterate(batch, 0)
    status, res, scale, k = None, (math.nan, math.nan, math.nan), 1.0, 1
    while status is None and k <= config.max_iter:
        K = 1 if k == 1 else min(KMAX, config.max_iter - k + 1)
        if callback is not None and k > 1:
            K = min(K, config.progress_every - (k - 1) % config.progress_every)
        conv = config.eps_tol * scale if k > 1 else -1.0
        if dense:
            outs, done = [[batch.iterate_dense(0, n, it.ypar)]], [1]
        else:
            outs, done = batch.iterate_many([0], [n], [it.ypar], K, [conv], np.full(K, np.inf))
        for j in range(int(done[0])):
            out = outs[0][j]
            if out[OUT_FINITE] != 1.0:                   # pdhg.py:251-253
                status = SolveStatus.DIVERGED
                it.which = 1
                break
            it.k = k
            it.ypar ^= 1
            it.which = 0
            ep, ed = float(out[OUT_EPS_P]), float(out[OUT_EPS_D])
            res = (ep, ed, ep + ed)
            if k == 1 and config.relative_residuals:
                scale = 1.0 + res[2]
            if callback is not None and k % config.progress_every == 0:
                callback(ProgressInfo(k, *res, n, it.objective()))
            k += 1
            if res[2] <= config.eps_tol * scale:
                status = SolveStatus.OPTIMAL
                break
        if status is None and time.perf_counter() - t0 > config.time_limit_s:
            status = SolveStatus.TIME_LIMIT
    if status is None:
        status = SolveStatus.MAX_ITERATIONS
    X, y = it.X(), it.y()
    pobj = prob.C.inner(X)
    dobj = -float(prob.b @ y[: prob.m] + prob.h @ y[prob.m:])
    return SolveResult(status=status, X=X, y=y, primal_objective=pobj, dual_objective=dobj,
                       final_residuals=res, iterations=it.k, rank_path=[(0, n)], checkpoints=[],
                       wall_time_s=time.perf_counter() - t0, residual_scale=scale,
                       objective_sign=prob.objective_sign)


def check_solution(prob: SdpProblem, X: SymMatrix, y, tol: float = 1e-3) -> SolutionReport:
    """Objectives, constraint violations, minimum eigenvalue and duality gap
    (reference ``problem.py:213-240``).  A(X) runs on the device; the minimum
    eigenvalue comes from the device eigensolver instead of a dense O(n^3)
    ``eigvalsh``: lambda_min(X) = c - lambda_max(c I - X) with c above the
    Gershgorin bound of X, lambda_max read off the rank-1 projection."""
    from .device import aproj_psd_packed
    from .layout import packed_coords
    prob = as_problem(prob)
    y = np.asarray(y, dtype=float)
    if X.n != prob.n or y.shape != (prob.m + prob.p,):
        raise ValueError("solution dimensions do not match the problem")
    mx = _device_batch(prob).apply_M(0, X.data)
    eq = float(np.linalg.norm(mx[: prob.m] - prob.b))
    ineq = float(np.linalg.norm(np.maximum(mx[prob.m:] - prob.h, 0.0)))
    pobj = prob.C.inner(X)
    dobj = -float(prob.b @ y[: prob.m] + prob.h @ y[prob.m:])
    n = X.n
    i, j = packed_coords(n, np.arange(X.data.size))
    diag = i == j
    dense_abs = np.where(diag, np.abs(X.data), np.abs(X.data) / math.sqrt(2.0))
    rowsum = np.bincount(i, dense_abs, minlength=n) + np.bincount(j[~diag], dense_abs[~diag], minlength=n)
    c = float(rowsum.max()) + 1.0
    S = -X.data.copy()
    S[diag] += c
    if n == 1:
        lam_max = float(S[0])
    else:
        P, _ = aproj_psd_packed(n, S, 1)
        lam_max = float(np.sum(P[diag]))
    min_eig = c - lam_max
    report = SolutionReport(primal_objective=pobj, dual_objective=dobj, equality_violation=eq,
                            inequality_violation=ineq, min_eigenvalue=min_eig, duality_gap=pobj - dobj)
    if report.max_violation() > tol:
        logger.debug("solution violates constraints beyond tol=%.1e (max violation %.3e)",
                     tol, report.max_violation())
    return report
