"""Multi-process (world_size 2, gloo on CPU) checks of the sharding + record all-gather logic."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1805_09258_b200.dist import build_records_sharded, shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def fake_builder(scene, X, seeds):
    """CPU stand-in for the GPU build: a deterministic function of (point, seed words)."""
    n = X.shape[0]
    out = np.zeros((n, 2, 7))
    out[:, 0, :3] = X
    out[:, 1, :3] = seeds.astype(np.float64)
    out[:, :, 6] = X.sum(axis=1, keepdims=True)
    return torch.tensor(out)


def _worker(rank, world, port, N, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    X = np.random.default_rng(0).uniform(0, 1, (N, 3))
    recs, (lo, hi) = build_records_sharded(None, X, 2, builder=fake_builder)
    q.put((rank, lo, hi, recs.numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("N", [7, 16, 1])
def test_sharded_build_and_all_gather_world2(N):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, N, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    X = np.random.default_rng(0).uniform(0, 1, (N, 3))
    from paper_1805_09258_b200.records import seed_words

    ref = fake_builder(None, X, seed_words(2, 401, np.arange(N))).numpy()
    shards = sorted((r, lo, hi) for r, lo, hi, _ in got)
    assert shards[0][1] == 0 and shards[-1][2] == N and shards[0][2] == shards[1][1]
    for _, _, _, recs in got:
        np.testing.assert_array_equal(recs, ref)  # every rank holds all records, global order


def test_shard_range_partitions():
    for n in (0, 1, 5, 19000):
        for w in (1, 2, 3, 8):
            r = [shard_range(n, k, w) for k in range(w)]
            assert r[0][0] == 0 and r[-1][1] == n
            assert all(r[k][1] == r[k + 1][0] for k in range(w - 1))
            sizes = [b - a for a, b in r]
            assert max(sizes) - min(sizes) <= 1
