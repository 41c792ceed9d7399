"""Op-level drop-ins for the reference's linear maps and truncated PSD
projection, each one call into the sm_100a library.

* ``apply_M``          reference ``problem.py:140-144``
* ``apply_M_adjoint``  reference ``problem.py:147-154``
* ``aproj_psd``        reference ``symmat.py:229-245`` (device eigensolver)
"""

from __future__ import annotations

import numpy as np

from .device import aproj_psd_packed
from .layout import SymMatrix
from .model import SdpProblem, as_problem
from .solver import _device_batch


def apply_M(prob: SdpProblem, X: SymMatrix) -> np.ndarray:
    prob = as_problem(prob)
    if X.n != prob.n:
        raise ValueError(f"matrix dimension {X.n} does not match problem {prob.n}")
    return _device_batch(prob).apply_M(0, X.data)


def apply_M_adjoint(prob: SdpProblem, y) -> SymMatrix:
    prob = as_problem(prob)
    y = np.asarray(y, dtype=float)
    if y.shape != (prob.m + prob.p,):
        raise ValueError(f"multiplier length {y.size} does not match m+p={prob.m + prob.p}")
    return SymMatrix(prob.n, _device_batch(prob).apply_M_adjoint(0, y))


def aproj_psd(S: SymMatrix, r: int) -> tuple[SymMatrix, float]:
    if not 1 <= r <= S.n:
        raise ValueError(f"rank r={r} outside [1, {S.n}]")
    P, lam = aproj_psd_packed(S.n, S.data, r)
    return SymMatrix(S.n, P), float(lam)
