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


def _render_worker(rank, world, port, H, W, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from types import SimpleNamespace

    from paper_1805_09258_b200.dist import broadcast_cache_set, render_sharded
    from paper_1805_09258_b200.records import record_size
    from paper_1805_09258_b200.cache import RadianceCache

    bmin, bmax = np.zeros(3), np.ones(3)
    cs = SimpleNamespace(single=RadianceCache(bmin, bmax), multiple=RadianceCache(bmin, bmax))
    if rank == 0:  # only rank 0 populated; the others start empty
        rows = np.random.default_rng(5).uniform(0.1, 0.9, (7, record_size(3)))
        cs.single.extend_packed(rows)
        cs.multiple.extend_packed(rows[:3] * 2)
    broadcast_cache_set(cs)
    camera = SimpleNamespace(height=H, width=W)
    settings = SimpleNamespace(frozen=True, mode="ours-aniso")

    def fake_rows(scene, cam, st, cache_set, row0, rows):
        """CPU stand-in for the device march: a function of the global pixel and the records."""
        r = np.arange(row0, row0 + rows)[:, None, None]
        c = np.arange(cam.width)[None, :, None]
        k = cache_set.single.packed().sum() + 10 * cache_set.multiple.packed().sum()
        slab = (r * 1000 + c) + np.arange(3)[None, None, :] * 0.25 + k
        return slab, {"cache_hits": rows * cam.width, "direct_evaluations": rows}

    img, st = render_sharded(None, camera, settings, cs, renderer=fake_rows)
    q.put((rank, img, st, cs.single.packed(), cs.multiple.packed()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("H", [5, 1])
def test_render_sharded_world2(H):
    """Row-sharded frozen render: rank 0's records reach every rank, row slabs reassemble
    into the full image in row order on every rank, and the counts sum."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    W = 4
    procs = [ctx.Process(target=_render_worker, args=(r, 2, port, H, W, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = sorted((q.get(timeout=120) for _ in range(2)), key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    from paper_1805_09258_b200.records import record_size

    rows = np.random.default_rng(5).uniform(0.1, 0.9, (7, record_size(3)))
    k = rows.sum() + 10 * (rows[:3] * 2).sum()
    want = (np.arange(H)[:, None, None] * 1000 + np.arange(W)[None, :, None]) + np.arange(3) * 0.25 + k
    for rank, img, st, ps, pm in got:
        np.testing.assert_array_equal(ps, rows)
        np.testing.assert_array_equal(pm, rows[:3] * 2)
        np.testing.assert_allclose(img, want, rtol=0, atol=1e-9)
        assert st["cache_hits"] == H * W and st["direct_evaluations"] == H


def _wave_worker(rank, world, port, sizes, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1805_09258_b200.dist import all_gather_rows, sharded_wave

    out = []
    for n in sizes:
        X = np.random.default_rng(n).uniform(0, 1, (n, 3))
        words = np.stack([np.full(n, 5), np.full(n, 401), np.arange(n)], axis=1).astype(np.uint32)
        built = []

        def build_local(lo, hi):
            built.append((lo, hi))
            recs = fake_builder(None, X[lo:hi], words[lo:hi]).reshape(hi - lo, 14)
            stats = torch.tensor(np.stack([np.arange(lo, hi), np.zeros(hi - lo, np.int64)], axis=1))
            return torch.cat([recs, stats.view(torch.float64)], dim=1)

        rows = sharded_wave(n, build_local, lambda t: all_gather_rows(t), rank, world)
        out.append((n, built[0], rows.numpy()))
    q.put((rank, out))
    dist.barrier()
    dist.destroy_process_group()


def test_populate_wave_sharding_world2():
    """The multi-GPU populate's per-wave exchange (dist.populate_sharded → sharded_wave): each
    rank builds a contiguous share of the wave's points and the all-gather hands every rank
    the rows of the whole wave in wave order, equal to one rank building the whole wave —
    so every rank's engine resolves identical records (waves smaller than the world
    included)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    sizes = [5, 1, 0, 64, 2]
    procs = [ctx.Process(target=_wave_worker, args=(r, 2, port, sizes, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = sorted((q.get(timeout=120) for _ in range(2)), key=lambda t: t[0])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for k, n in enumerate(sizes):
        X = np.random.default_rng(n).uniform(0, 1, (n, 3))
        words = np.stack([np.full(n, 5), np.full(n, 401), np.arange(n)], axis=1).astype(np.uint32)
        want = fake_builder(None, X, words).reshape(n, 14).numpy()
        shares = [got[r][1][k][1] for r in range(2)]
        assert shares[0][0] == 0 and shares[0][1] == shares[1][0] and shares[1][1] == n
        for r in range(2):
            rows = got[r][1][k][2]
            assert rows.shape[0] == n
            np.testing.assert_array_equal(rows[:, :want.shape[1]], want)
            np.testing.assert_array_equal(rows[:, want.shape[1]:].copy().view(np.int64)[:, 0], np.arange(n))
