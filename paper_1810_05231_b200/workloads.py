"""Seeded synthetic workloads for the five BASELINE.json configurations.

The reference ships no Max-Cut generator and its equipartition / sensor
generators differ from the BASELINE configs, so the
recipes are frozen here.  Every builder returns the drop-in
:class:`~.model.SdpProblem` plus the :class:`~.config.SolverConfig` the config
is quoted with.

Graph recipe (configs 1, 2, 3, 5): ``rng = default_rng(seed)``; candidate
pairs ``triu_indices(n, 1)`` (the ``itertools.combinations`` order of the
reference's ``random_graph``, ``instances.py:129-139``); ``keep = rng.random
< p``; +-1 weights from the next draw ``where(rng.random(|E|) < 0.5, -1, 1)``
(mirrors ``instances.py:195``).  Laplacian ``L = diag(W 1) - W``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .config import SolverConfig
from .layout import SQRT2, SymMatrix, packed_length, row_starts
from .model import SdpProblem, SparseRow


@dataclass
class GraphEdges:
    n: int
    i: np.ndarray
    j: np.ndarray
    w: np.ndarray


def random_graph(n: int, p: float, seed: int, signed: bool) -> GraphEdges:
    rng = np.random.default_rng(seed)
    iu, ju = np.triu_indices(n, 1)
    keep = rng.random(iu.size) < p
    i, j = iu[keep], ju[keep]
    if signed:
        w = np.where(rng.random(i.size) < 0.5, -1.0, 1.0)
    else:
        w = np.ones(i.size)
    return GraphEdges(n, i.astype(np.int64), j.astype(np.int64), w)


def laplacian_packed(g: GraphEdges, scale: float) -> np.ndarray:
    """svec(scale * L) built directly in packed form (no dense n x n)."""
    n = g.n
    out = np.zeros(packed_length(n))
    deg = np.zeros(n)
    np.add.at(deg, g.i, g.w)
    np.add.at(deg, g.j, g.w)
    starts = row_starts(n)
    out[starts] = scale * deg
    # off-diagonal packed entries: -scale * w * sqrt(2); edges are unique pairs
    out[starts[g.i] + (g.j - g.i)] = -scale * g.w * SQRT2
    return out


def diag_pin_rows(n: int) -> list:
    starts = row_starts(n)
    return [SparseRow(np.array([s]), np.array([1.0])) for s in starts]


def maxcut_problem(n: int, p: float, seed: int, signed: bool) -> SdpProblem:
    """min <-L/4, X>  s.t. diag(X) = 1,  X psd."""
    g = random_graph(n, p, seed, signed)
    return SdpProblem(
        n=n,
        C=SymMatrix(n, laplacian_packed(g, -0.25)),
        A=diag_pin_rows(n),
        b=np.ones(n),
        name=f"maxcut_n{n}_p{p}_s{seed}",
    )


def equipartition_problem(n: int, p: float, seed: int) -> SdpProblem:
    """min <L/4, X> s.t. diag(X) = 1, <11^T, X> = 0, X psd (one dense row)."""
    g = random_graph(n, p, seed, signed=False)
    P = packed_length(n)
    ones = np.full(P, SQRT2)
    ones[row_starts(n)] = 1.0
    rows = diag_pin_rows(n) + [SparseRow(np.arange(P, dtype=np.int64), ones)]
    return SdpProblem(
        n=n,
        C=SymMatrix(n, laplacian_packed(g, 0.25)),
        A=rows,
        b=np.concatenate([np.ones(n), [0.0]]),
        name=f"equipartition_n{n}_p{p}_s{seed}",
    )


SENSOR_ANCHORS = np.array([[-0.45, -0.45], [-0.45, 0.45], [0.45, -0.45], [0.45, 0.45]])


def sensor_problem(n_sensors: int = 1000, radius: float = 0.1, seed: int = 0,
                   trace_reg: float = 1e-3) -> SdpProblem:
    """Biswas-Ye localisation over Z = [[I_2, X], [X^T, Y]] (d = 2).

    Same row construction as the reference's ``gen_sensor_localization``
    (``instances.py:262-315``): identity-block pins, one row per measured
    sensor pair (Y_ii + Y_jj - 2Y_ij = w^2) and one per anchor-sensor pair
    ([a; -e_j][a; -e_j]^T).  Noise-free distances within ``radius``; objective
    ``trace_reg * tr(Z)``.
    """
    d = 2
    rng = np.random.default_rng(seed)
    sensors = rng.random((n_sensors, d)) - 0.5
    nz = d + n_sensors
    rows, rhs = [], []
    for a in range(d):
        for c in range(a, d):
            rows.append(SparseRow.from_matrix_entries(nz, [(a, c, 1.0 if a == c else 0.5)]))
            rhs.append(1.0 if a == c else 0.0)
    iu, ju = np.triu_indices(n_sensors, 1)
    dist = np.linalg.norm(sensors[iu] - sensors[ju], axis=1)
    sel = dist <= radius
    for i, j, w in zip(iu[sel], ju[sel], dist[sel]):
        rows.append(SparseRow.from_matrix_entries(
            nz, [(d + i, d + i, 1.0), (d + j, d + j, 1.0), (d + i, d + j, -1.0)]))
        rhs.append(float(w) ** 2)
    for k in range(SENSOR_ANCHORS.shape[0]):
        ak = SENSOR_ANCHORS[k]
        dk = np.linalg.norm(sensors - ak, axis=1)
        for j in np.nonzero(dk <= radius)[0]:
            ent = [(a, c, ak[a] * ak[c]) for a in range(d) for c in range(a, d)]
            ent += [(a, d + int(j), -ak[a]) for a in range(d)]
            ent.append((d + int(j), d + int(j), 1.0))
            rows.append(SparseRow.from_matrix_entries(nz, ent))
            rhs.append(float(dk[j]) ** 2)
    C = np.zeros(packed_length(nz))
    C[row_starts(nz)] = trace_reg
    return SdpProblem(n=nz, C=SymMatrix(nz, C), A=rows, b=np.array(rhs),
                      name=f"sensor_s{n_sensors}_r{radius}")


BIG_TIME = 1e9


def config(idx: int, seed: int = 0):
    """(problem, SolverConfig) for BASELINE.json configs[idx] (0-based)."""
    if idx == 0:
        return maxcut_problem(100, 0.1, seed, signed=False), SolverConfig(
            eps_tol=1e-4, max_iter=2000, initial_rank=5)
    if idx == 1:
        return maxcut_problem(2000, 0.01, seed, signed=True), SolverConfig(
            eps_tol=1e-4, initial_rank=10, time_limit_s=BIG_TIME)
    if idx == 2:
        return equipartition_problem(5000, 0.002, seed), SolverConfig(
            eps_tol=1e-4, initial_rank=10, time_limit_s=BIG_TIME)
    if idx == 3:
        return sensor_problem(1000, 0.1, seed), SolverConfig(
            eps_tol=1e-4, time_limit_s=BIG_TIME)
    if idx == 4:
        return maxcut_problem(1000, 0.02, seed, signed=True), SolverConfig(
            eps_tol=1e-4, time_limit_s=BIG_TIME)
    raise ValueError(f"unknown config index {idx}")
