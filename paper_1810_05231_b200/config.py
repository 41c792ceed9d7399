"""Solver configuration, result types and the host-side rank controller.

These are the reference's public result/config types with identical fields,
defaults and validation messages (``pkg/src/pdsdp/pdhg.py:32-140`` and
``pkg/src/pdsdp/lowrank.py:39-83``).  The rank-adaptation and stopping logic
stays on the host, exactly as the north star asks; only scalars cross from
the device per iteration.
"""

from __future__ import annotations

from collections import deque
from dataclasses import dataclass, field
from enum import Enum
from typing import Callable, NamedTuple

import numpy as np

from .layout import SymMatrix, approx_error_bound


class SolveStatus(Enum):
    """Run outcome (reference ``pdhg.py:32-36``).  Members compare and hash
    equal to the same-named members of any other ``SolveStatus`` enum with
    the same value, so tables keyed by the reference's own members (its
    ``cli._status_exit_code``, ``cli.py:178-186``) accept results of this
    package without importing either side into the other."""

    OPTIMAL = "optimal"
    MAX_ITERATIONS = "max_iterations"
    TIME_LIMIT = "time_limit"
    DIVERGED = "diverged"

    def __eq__(self, other):
        if self is other:
            return True
        if isinstance(other, Enum) and type(other).__name__ == "SolveStatus":
            return other.name == self.name and other.value == self.value
        return NotImplemented

    def __hash__(self):
        return hash(self._name_)      # Enum's own hash: same bucket as the reference member


# eps_lambda defaults to this times n (reference pdhg.py:39)
DEFAULT_EPS_LAMBDA_PER_N = 5e-2


@dataclass
class SolverConfig:
    """Tolerances, step size policy and limits (reference ``pdhg.py:42-85``)."""

    eps_tol: float = 1e-3
    eps_lambda: float | None = None
    alpha_safety: float = 0.99
    window_ell: int = 500
    max_iter: int = 100_000
    time_limit_s: float = 1200.0
    seed: int = 0
    initial_rank: int = 1
    relative_residuals: bool = True
    alpha_override: float | None = None
    progress_every: int = 100

    def validate(self) -> None:
        checks = (
            (self.eps_tol <= 0, "eps_tol must be positive"),
            (not 0 < self.alpha_safety < 1, "alpha_safety must lie in (0, 1)"),
            (self.window_ell < 1, "window_ell must be at least 1"),
            (self.max_iter < 1, "max_iter must be at least 1"),
            (self.time_limit_s <= 0, "time_limit_s must be positive"),
            (self.initial_rank < 1, "initial_rank must be at least 1"),
            (self.eps_lambda is not None and self.eps_lambda < 0,
             "eps_lambda must be nonnegative"),
            (self.alpha_override is not None and self.alpha_override <= 0,
             "alpha_override must be positive"),
            (self.progress_every < 1, "progress_every must be at least 1"),
        )
        for bad, msg in checks:
            if bad:
                raise ValueError(msg)


class ProgressInfo(NamedTuple):
    """Callback snapshot (reference ``pdhg.py:88-96``)."""

    k: int
    eps_primal: float
    eps_dual: float
    eps_comb: float
    rank: int
    objective: float


ProgressCallback = Callable[[ProgressInfo], None]


@dataclass
class SolveResult:
    """Solve outcome (reference ``pdhg.py:121-140``)."""

    status: SolveStatus
    X: SymMatrix
    y: np.ndarray
    primal_objective: float
    dual_objective: float
    final_residuals: tuple
    iterations: int
    rank_path: list
    checkpoints: list = field(default_factory=list)
    wall_time_s: float = 0.0
    residual_scale: float = 1.0
    objective_sign: float = 1.0

    @property
    def reported_objective(self) -> float:
        return self.objective_sign * self.primal_objective


@dataclass
class SolutionReport:
    """Feasibility and optimality summary of a primal-dual pair (reference
    ``problem.py:186-210``)."""

    primal_objective: float
    dual_objective: float
    equality_violation: float
    inequality_violation: float
    min_eigenvalue: float
    duality_gap: float

    def max_violation(self) -> float:
        return max(self.equality_violation, self.inequality_violation, -min(self.min_eigenvalue, 0.0))


@dataclass
class Checkpoint:
    """Feasible pair saved on inner convergence (reference ``lowrank.py:39-47``)."""

    rank: int
    X: SymMatrix
    y: np.ndarray
    objective: float = 0.0


@dataclass
class RankController:
    """Target rank, stall window, saved pairs (reference ``lowrank.py:50-61``)."""

    r: int
    ell: int
    history: deque = field(default_factory=deque)
    checkpoints: list = field(default_factory=list)
    last_lambda_r: float = float("inf")

    def __post_init__(self):
        self.history = deque(self.history, maxlen=self.ell + 1)


def stall_detected(history, ell: int) -> bool:
    """Newest combined residual no better than the one ``ell`` back
    (reference ``lowrank.py:64-69``)."""
    return len(history) >= ell + 1 and history[-1] >= history[-1 - ell]


def update_rank(controller: RankController, n: int) -> int:
    """r <- min(2r, n), clear the window (reference ``lowrank.py:72-76``)."""
    controller.r = min(2 * controller.r, n)
    controller.history.clear()
    return controller.r


def rank_certificate_satisfied(n: int, r: int, lambda_r: float, eps_lambda: float) -> bool:
    """(n - r) max(lambda_{r+1}, 0) <= eps_lambda (reference ``lowrank.py:79-83``)."""
    return approx_error_bound(n, r, lambda_r) <= eps_lambda
