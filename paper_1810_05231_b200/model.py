"""Problem data model of the general-form SDP (host side, drop-in types).

    min tr(CX)  s.t.  tr(A_i X) = b_i,  tr(G_j X) <= h_j,  X psd

Same fields, validation and error messages as the reference data model
(``pkg/src/pdsdp/problem.py:29-137``): ``C`` is a packed :class:`SymMatrix`,
each constraint is a :class:`SparseRow` of its packed form (strictly
increasing int64 positions, sqrt(2)-scaled off-diagonal values).  The device
never sees this layout inside the loop; :mod:`.device` re-indexes it once
into dense (i, j) coordinates when a problem is uploaded.
"""

from __future__ import annotations

import weakref
from dataclasses import dataclass, field

import numpy as np

from .layout import SQRT2, SymMatrix, packed_index, packed_length


@dataclass
class SparseRow:
    """One constraint matrix as sparse packed entries
    (reference ``problem.py:29-70``)."""

    indices: np.ndarray
    values: np.ndarray

    def __post_init__(self):
        self.indices = np.asarray(self.indices, dtype=np.int64)
        self.values = np.asarray(self.values, dtype=float)
        if self.indices.shape != self.values.shape or self.indices.ndim != 1:
            raise ValueError("indices and values must be 1-d of equal length")
        if self.indices.size and np.any(np.diff(self.indices) <= 0):
            raise ValueError("indices must be strictly increasing")
        if self.indices.size and self.indices[0] < 0:
            raise ValueError("negative packed index")
        if not np.all(np.isfinite(self.values)):
            raise ValueError("non-finite constraint value")

    @classmethod
    def from_matrix_entries(cls, n: int, entries) -> "SparseRow":
        """(i, j, value) matrix entries with i <= j; duplicates summed
        (reference ``problem.py:52-66``)."""
        acc: dict[int, float] = {}
        for i, j, v in entries:
            pos = packed_index(n, i, j)
            acc[pos] = acc.get(pos, 0.0) + (1.0 if i == j else SQRT2) * float(v)
        keys = sorted(acc)
        return cls(np.array(keys, dtype=np.int64), np.array([acc[k] for k in keys]))

    def dot_packed(self, data) -> float:
        return float(self.values @ np.asarray(data)[self.indices])


@dataclass
class SdpProblem:
    """Immutable-by-convention problem data (reference ``problem.py:73-137``)."""

    n: int
    C: SymMatrix
    A: list
    b: np.ndarray
    G: list = field(default_factory=list)
    h: np.ndarray = field(default_factory=lambda: np.zeros(0))
    name: str = ""
    objective_sign: float = 1.0

    def __post_init__(self):
        self.b = np.asarray(self.b, dtype=float)
        self.h = np.asarray(self.h, dtype=float)
        if self.C.n != self.n:
            raise ValueError("objective matrix dimension mismatch")
        if len(self.A) != self.b.size or len(self.G) != self.h.size:
            raise ValueError("constraint row/right-hand-side count mismatch")
        if len(self.A) + len(self.G) < 1:
            raise ValueError("problem needs at least one constraint")
        if not (np.all(np.isfinite(self.b)) and np.all(np.isfinite(self.h))):
            raise ValueError("non-finite right-hand side")
        if not np.all(np.isfinite(self.C.data)):
            raise ValueError("non-finite objective data")
        plen = packed_length(self.n)
        for row in list(self.A) + list(self.G):
            if row.indices.size and row.indices[-1] >= plen:
                raise ValueError("constraint row index out of range")
        self._csr = None
        self._device_cache = {}

    @property
    def m(self) -> int:
        return len(self.A)

    @property
    def p(self) -> int:
        return len(self.G)

    @property
    def packed_len(self) -> int:
        return packed_length(self.n)

    def stacked_arrays(self):
        """(indptr int64[m+p+1], indices int64[nnz], values float64[nnz]) of
        the stacked operator M = [A; G] over packed positions — the CSR the
        reference builds in ``problem.py:119-137``, without scipy."""
        if self._csr is None:
            rows = list(self.A) + list(self.G)
            indptr = np.zeros(len(rows) + 1, dtype=np.int64)
            indptr[1:] = np.cumsum([r.indices.size for r in rows])
            idx = np.concatenate([r.indices for r in rows]) if rows else np.zeros(0, np.int64)
            val = np.concatenate([r.values for r in rows]) if rows else np.zeros(0)
            self._csr = (indptr, idx.astype(np.int64), val.astype(float))
        return self._csr


# Reference-typed problems (``pdsdp.SdpProblem``, reference ``problem.py:74-137``)
# are accepted wherever this package takes a problem: they are read by duck
# typing (n, C.data, the rows' indices / values, b, h, objective_sign) -- the
# reference package is never imported -- and the converted problem, which owns
# the device cache, is kept off-object for as long as the caller's object lives.
_converted: dict = {}


def as_problem(prob) -> "SdpProblem":
    """This package's :class:`SdpProblem` for ``prob``: ``prob`` itself, or the
    cached field-by-field conversion of any object laid out like the
    reference's ``SdpProblem`` (``problem.py:74-87``)."""
    if isinstance(prob, SdpProblem):
        return prob
    key = id(prob)
    hit = _converted.get(key)
    if hit is not None and hit[0]() is prob:
        return hit[1]
    try:
        conv = SdpProblem(
            n=int(prob.n),
            C=SymMatrix(int(prob.C.n), np.asarray(prob.C.data, dtype=float)),
            A=[SparseRow(r.indices, r.values) for r in prob.A],
            b=np.asarray(prob.b, dtype=float),
            G=[SparseRow(r.indices, r.values) for r in getattr(prob, "G", [])],
            h=np.asarray(getattr(prob, "h", np.zeros(0)), dtype=float),
            name=str(getattr(prob, "name", "")),
            objective_sign=float(getattr(prob, "objective_sign", 1.0)),
        )
    except AttributeError as exc:
        raise TypeError(f"not an SdpProblem-like object: {exc}") from None
    try:
        ref = weakref.ref(prob, lambda _r, k=key: _converted.pop(k, None))
    except TypeError:                     # object without weakref support: convert every time
        return conv
    _converted[key] = (ref, conv)
    return conv
