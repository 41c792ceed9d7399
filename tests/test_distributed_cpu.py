"""Multi-rank host logic on CPU: world_size 2 over gloo (no GPU)."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_1810_05231_b200.distributed import FIELDS, gather_summaries, shard


def test_shard_partition_is_exact():
    for count in (1, 7, 256):
        for world in (1, 2, 3, 8):
            seen = [i for q in range(world) for i in shard(count, q, world)]
            assert seen == list(range(count))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, count, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    mine = shard(count, rank, world)
    local = np.array([[i, -i, 0.1 * i, 0.2 * i, 0.3 * i, 100 + i, 2, 0] for i in mine], dtype=float)
    local = local.reshape(-1, len(FIELDS))
    full = gather_summaries(local, count, rank, world)
    q.put((rank, full))
    dist.destroy_process_group()


@pytest.mark.parametrize("count", [5, 8])
def test_gather_summaries_two_ranks_gloo(count):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, count, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, full in got:
        assert full.shape == (count, len(FIELDS))
        np.testing.assert_array_equal(full[:, 0], np.arange(count))
        np.testing.assert_array_equal(full[:, 5], 100 + np.arange(count))


def test_bench_gpus_flag_spawns_ranks():
    """`python bench.py --gpus 2` without a launcher re-executes itself under
    torch.distributed.run (one process per GPU) and prints ONE JSON line with
    n_gpus = 2 (CPU check of the launcher path: gloo, no CUDA work)."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--launcher-check"],
                         capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == 2 and rec["ranks"] == [0, 1]
