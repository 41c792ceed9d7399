"""Host-side Algorithm-2 logic on CPU (no GPU): the bulk fold of uneventful
chunk steps must leave exactly the state the step-by-step replay of the
reference's control flow (lowrank.py:141-188) leaves; the reference arm's rank
shares come from rank paths."""

import numpy as np

from paper_1810_05231_b200 import workloads
from paper_1810_05231_b200.config import SolverConfig
from paper_1810_05231_b200.device import OUT_EIGCONV, OUT_EPS_D, OUT_EPS_P, OUT_FINITE, OUT_LAMBDA, OUT_LEN, \
    OUT_MATVECS, OUT_PASSES
from paper_1810_05231_b200.solver import _InstanceRun


class _StubBatch:
    """Just enough of DeviceBatch for _InstanceRun without a device."""

    def __init__(self, prob):
        self.problems = [prob]

    def set_alpha(self, inst, alpha):
        pass

    def reset(self, inst, seed=0.0):
        pass


def _chunk(rng, K, level, stall_at=None):
    out = np.zeros((K, OUT_LEN))
    ec = level * (1.0 - 1e-3 * np.arange(1, K + 1)) * (1.0 + 1e-6 * rng.standard_normal(K))
    out[:, OUT_EPS_P] = 0.7 * ec
    out[:, OUT_EPS_D] = 0.3 * ec
    out[:, OUT_LAMBDA] = rng.standard_normal(K)
    out[:, OUT_FINITE] = 1.0
    out[:, OUT_PASSES] = rng.integers(1, 4, K)
    out[:, OUT_MATVECS] = rng.integers(3, 12, K)
    out[:, OUT_EIGCONV] = 1.0
    if stall_at is not None:
        out[stall_at, OUT_EPS_P] *= 50.0        # a residual bump: the stall rule fires at this step
    return out


def _state(run):
    c = run.controller
    return (run.k, run.it.k, run.it.ypar, run.it.which, run.res, run.scale, list(c.history), c.r,
            c.last_lambda_r, list(run.rank_path), run.eig_passes, run.eig_matvecs, run.eig_unconverged, run.status)


def test_bulk_fold_matches_stepwise_replay():
    prob = workloads.maxcut_problem(40, 0.2, 1, signed=True)
    cfg = SolverConfig(eps_tol=1e-9, initial_rank=2, window_ell=20, max_iter=10_000)
    rng = np.random.default_rng(5)
    runs = [_InstanceRun(_StubBatch(prob), 0, prob, cfg, 0.5, None, 0.0) for _ in range(2)]
    # first iteration alone (it fixes the relative scale), then chunks; the
    # last step of the third chunk trips the stall rule (window_ell = 20)
    first = _chunk(rng, 1, 5.0)
    chunks = [first, _chunk(rng, 16, 4.0), _chunk(rng, 16, 3.5), _chunk(rng, 16, 3.0, stall_at=15),
              _chunk(rng, 7, 2.5), _chunk(rng, 16, 2.0)]
    for out in chunks:
        runs[0].consume(out, len(out))                 # bulk fold + last step
        runs[1]._consume_steps(out, 0, len(out))        # the reference's loop, step by step
        assert _state(runs[0]) == _state(runs[1])
    assert runs[0].rank_path == [(0, 2), (49, 4)]      # the stall fired exactly at the bumped step
    assert runs[0].k == 1 + 16 * 4 + 7 + 1


def test_bulk_fold_refuses_eventful_steps():
    """A chunk whose inner steps hold an event (the device would have paused
    there) must not be folded: the guard sends it down the stepwise path."""
    prob = workloads.maxcut_problem(30, 0.2, 2, signed=True)
    cfg = SolverConfig(eps_tol=1e-9, initial_rank=2, window_ell=12, max_iter=10_000)   # chunks never exceed the window (max_chunk)
    rng = np.random.default_rng(6)
    run = _InstanceRun(_StubBatch(prob), 0, prob, cfg, 0.5, None, 0.0)
    run.consume(_chunk(rng, 1, 5.0), 1)
    run.consume(_chunk(rng, 12, 4.0), 12)
    bumped = _chunk(rng, 12, 3.5, stall_at=4)           # event in the middle
    assert not run._bulk_ok(bumped, 11)
    nonfinite = _chunk(rng, 12, 3.0)
    nonfinite[3, OUT_FINITE] = 0.0
    assert not run._bulk_ok(nonfinite, 11)


def test_rank_shares_from_rank_path():
    import bench
    sh = bench.rank_shares(99, fallback=([(0, 10), (750, 20)], 1000))
    assert sh == {10: 0.75, 20: 0.25}
    sh = bench.rank_shares(1)                            # fixture or the measured path of config 2
    assert abs(sum(sh.values()) - 1.0) < 1e-12 and set(sh) == {10, 20}


def test_unfinished_step_switches_the_instance_to_the_dense_path():
    """A chunk that reports a step needing more than an eigen block (output slot
    13) counts the steps before it and continues on the dense path from the
    same (X_k, y_k) -- the reference's dense fallback, symmat.py:181-185."""
    from paper_1810_05231_b200.device import OUT_ERR

    class Stub(_StubBatch):
        def __init__(self, prob):
            super().__init__(prob)
            self.dense_calls = []

        def dense_begin(self, inst, from_factored):
            self.dense_calls.append((inst, from_factored))

    prob = workloads.maxcut_problem(40, 0.2, 1, signed=True)
    cfg = SolverConfig(eps_tol=1e-9, initial_rank=2, window_ell=50, max_iter=10_000)
    rng = np.random.default_rng(7)
    batch = Stub(prob)
    run = _InstanceRun(batch, 0, prob, cfg, 0.5, None, 0.0)
    run.after_chunk(_chunk(rng, 1, 5.0), 1, 1)
    out = _chunk(rng, 16, 4.0)
    out[9, OUT_ERR] = 1.0                     # step 9 did not complete
    run.after_chunk(out, 9, 16)
    assert run.k == 1 + 1 + 9 - 1 + 1 and run.it.k == 10
    assert run.dense and batch.dense_calls == [(0, True)] and run.dense_from == run.k


def test_guard_columns_grow_at_rank_changes_of_many_pass_phases():
    prob = workloads.maxcut_problem(40, 0.2, 1, signed=True)
    cfg = SolverConfig(eps_tol=1e-9, initial_rank=2, window_ell=12, max_iter=10_000)
    rng = np.random.default_rng(8)
    run = _InstanceRun(_StubBatch(prob), 0, prob, cfg, 0.5, None, 0.0)
    run.after_chunk(_chunk(rng, 1, 5.0), 1, 1)
    many = _chunk(rng, 12, 4.0)
    many[:, OUT_PASSES] = 5                   # a phase that keeps needing five passes
    run.after_chunk(many, 12, 12)
    assert run.guard == 0 and run.flags() == 0
    bump = _chunk(rng, 12, 3.5, stall_at=11)  # the stall rule doubles the rank here
    bump[:, OUT_PASSES] = 5
    run.after_chunk(bump, 12, 12)
    assert run.controller.r == 4 and run.guard == 2 and run.flags() == 2 << 8
    calm = _chunk(rng, 12, 3.0, stall_at=11)  # one-pass phase: no further growth
    calm[:, OUT_PASSES] = 1
    run.after_chunk(_chunk(rng, 12, 3.2), 12, 12)
    run.after_chunk(calm, 12, 12)
    assert run.controller.r == 8 and run.guard == 2
