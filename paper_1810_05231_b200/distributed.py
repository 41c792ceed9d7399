"""Sharding of independent SDP instances over the GPUs of one box.

A single instance does not shard at these sizes, so the only
multi-GPU path is batch data parallelism: rank q of N solves a contiguous
block of instances on its own GPU, and the per-instance scalars
[pobj, dobj, eps_p, eps_d, eps_c, iterations, final rank, status] are
gathered with one all_gather over NCCL (gloo on CPU in the tests).
"""

from __future__ import annotations

import numpy as np

from .config import SolveStatus

FIELDS = ("primal_objective", "dual_objective", "eps_p", "eps_d", "eps_c", "iterations",
          "final_rank", "status")
_STATUS = {s: i for i, s in enumerate(SolveStatus)}


def shard(count: int, rank: int, world: int) -> range:
    """Contiguous, balanced block of instance indices owned by `rank`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    lo = (count * rank) // world
    hi = (count * (rank + 1)) // world
    return range(lo, hi)


def summarize(results) -> np.ndarray:
    """Per-instance scalar rows (float64[len, 8]) of SolveResults."""
    rows = []
    for r in results:
        ep, ed, ec = r.final_residuals
        final_rank = r.rank_path[-1][1] if r.rank_path else 0
        rows.append([r.primal_objective, r.dual_objective, ep, ed, ec, float(r.iterations),
                     float(final_rank), float(_STATUS[r.status])])
    return np.asarray(rows, dtype=np.float64).reshape(-1, len(FIELDS))


def gather_summaries(local: np.ndarray, count: int, rank: int, world: int, device=None) -> np.ndarray:
    """All ranks' summaries in instance order (float64[count, 8]).

    Blocks are padded to the largest shard so that one all_gather suffices."""
    import torch
    import torch.distributed as dist

    width = len(FIELDS)
    cap = max(len(shard(count, q, world)) for q in range(world))
    buf = np.zeros((cap, width))
    buf[: local.shape[0]] = local
    t = torch.from_numpy(buf).to(device if device is not None else "cpu")
    parts = [torch.zeros_like(t) for _ in range(world)]
    dist.all_gather(parts, t)
    out = np.zeros((count, width))
    for q in range(world):
        rng = shard(count, q, world)
        out[rng.start:rng.stop] = parts[q].cpu().numpy()[: len(rng)]
    return out
