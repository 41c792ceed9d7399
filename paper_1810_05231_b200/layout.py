"""Packed symmetric-matrix layout shared with the reference (host side).

The reference keeps every symmetric matrix as its upper triangle read row by
row (== lower triangle column by column), off-diagonal entries scaled by
sqrt(2) so that the Euclidean dot of two packed vectors equals tr(AB)
(reference ``pkg/src/pdsdp/symmat.py:1-8,50-101``).  This module provides that
layout for the drop-in API.  Nothing here runs inside the solve loop: the
device keeps its iterates in factored / dense form and packs only at the
boundary (``pdsdp_pack_lowrank`` in ``include/pdsdp_b200.h``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

SQRT2 = math.sqrt(2.0)


def packed_length(n: int) -> int:
    """n(n+1)/2 (reference ``symmat.py:37-39``)."""
    return n * (n + 1) // 2


def side_length(length: int) -> int:
    """Inverse of :func:`packed_length`; ValueError if not triangular
    (reference ``symmat.py:42-47``)."""
    n = (math.isqrt(8 * int(length) + 1) - 1) // 2
    if n < 1 or packed_length(n) != length:
        raise ValueError(f"packed length {length} is not triangular")
    return n


def packed_index(n: int, i: int, j: int) -> int:
    """Position of entry (i, j), 0 <= i <= j < n (reference ``symmat.py:50-54``)."""
    if not 0 <= i <= j < n:
        raise ValueError(f"entry ({i}, {j}) outside upper triangle of size {n}")
    return i * n - (i * (i - 1)) // 2 + (j - i)


def row_starts(n: int) -> np.ndarray:
    """Packed position of each diagonal entry (i, i)."""
    i = np.arange(n, dtype=np.int64)
    return i * n - (i * (i - 1)) // 2


def packed_coords(n: int, pos) -> tuple[np.ndarray, np.ndarray]:
    """(i, j) of packed positions (reference ``symmat.py:57-63``)."""
    pos = np.asarray(pos, dtype=np.int64)
    starts = row_starts(n)
    i = np.searchsorted(starts, pos, side="right") - 1
    return i, pos - starts[i] + i


def svec(S, tol: float = 1e-12) -> np.ndarray:
    """Dense symmetric -> packed, rejecting asymmetry above ``tol`` relative
    to the largest entry (reference ``symmat.py:66-86``)."""
    S = np.asarray(S, dtype=float)
    if S.ndim != 2 or S.shape[0] != S.shape[1]:
        raise ValueError(f"expected a square matrix, got shape {S.shape}")
    n = S.shape[0]
    if n == 0:
        raise ValueError("empty matrix")
    skew = float(np.max(np.abs(S - S.T)))
    if skew > tol * max(1.0, float(np.max(np.abs(S)))):
        raise ValueError(f"input is not symmetric: max |S - S.T| = {skew:.3e}")
    iu, ju = np.triu_indices(n)
    out = 0.5 * (S[iu, ju] + S[ju, iu])
    out[iu != ju] *= SQRT2
    return out


def smat(v) -> np.ndarray:
    """Packed -> dense symmetric (reference ``symmat.py:89-101``)."""
    v = np.asarray(v, dtype=float)
    if v.ndim != 1:
        raise ValueError(f"expected a 1-d packed vector, got shape {v.shape}")
    n = side_length(v.size)
    iu, ju = np.triu_indices(n)
    vals = np.where(iu == ju, v, v / SQRT2)
    out = np.empty((n, n))
    out[iu, ju] = vals
    out[ju, iu] = vals
    return out


@dataclass
class SymMatrix:
    """Symmetric matrix held packed (reference ``symmat.py:104-142``)."""

    n: int
    data: np.ndarray

    def __post_init__(self):
        self.data = np.asarray(self.data, dtype=float)
        if self.n < 1:
            raise ValueError(f"matrix dimension must be positive, got {self.n}")
        if self.data.shape != (packed_length(self.n),):
            raise ValueError(
                f"packed data has length {self.data.size}, "
                f"expected {packed_length(self.n)} for n={self.n}"
            )

    @classmethod
    def zero(cls, n: int) -> "SymMatrix":
        return cls(n, np.zeros(packed_length(n)))

    @classmethod
    def from_dense(cls, S, tol: float = 1e-12) -> "SymMatrix":
        S = np.asarray(S, dtype=float)
        return cls(S.shape[0], svec(S, tol))

    def to_dense(self) -> np.ndarray:
        return smat(self.data)

    def inner(self, other: "SymMatrix") -> float:
        return float(self.data @ other.data)

    def norm(self) -> float:
        return float(np.linalg.norm(self.data))

    def copy(self) -> "SymMatrix":
        return SymMatrix(self.n, self.data.copy())


@dataclass
class EigenDecomposition:
    """Eigenpairs, values descending (reference ``symmat.py:145-155``)."""

    values: np.ndarray
    vectors: np.ndarray
    truncated_rank: int | str = "full"


def approx_error_bound(n: int, r: int, lambda_r: float) -> float:
    """(n - r) * max(lambda_r, 0) (reference ``symmat.py:248-253``)."""
    if not 1 <= r <= n:
        raise ValueError(f"rank r={r} outside [1, {n}]")
    return float((n - r) * max(lambda_r, 0.0))
