"""Multi-GPU plumbing: record shards per rank, record all-gather before lookup.

One process per GPU (torchrun).  Cache points are split into contiguous index
ranges; every record's RNG stream depends only on its global index
(SeedSequence([seed, 401, i]), src/renderer.py:317), so the records are identical
whatever the sharding.  The build has no data-path collective; the only exchange is
an all-gather of the finished (padded, fixed-size) record arrays before a lookup /
march pass.
"""

from __future__ import annotations

import numpy as np


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [lo, hi) share of n items for `rank` (sizes differ by at most one)."""
    base, rem = divmod(n, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def all_gather_rows(t, group=None):
    """All-gather a (n_r, ...) tensor with per-rank n_r into the rank-ordered concatenation.

    Counts are exchanged first, then every rank pads to the max count (fixed-size
    collective) and the padding is dropped on reassembly.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    n = torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device)
    counts = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(counts, n, group=group)
    counts = [int(c.item()) for c in counts]
    m = max(counts)
    pad = torch.zeros((m,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    pad[: t.shape[0]] = t
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([p[:c] for p, c in zip(parts, counts)], dim=0)


def build_records_sharded(scene, X, cfg_seed: int, *, builder=None, group=None, **kw):
    """Build this rank's shard of records, then all-gather every rank's records.

    Returns (records (N, 2, RS) in global index order, this rank's [lo, hi)).
    `builder(scene, X_shard, seeds) -> (n, 2, RS) tensor` defaults to the GPU build;
    tests substitute a CPU stand-in to exercise the collective logic with gloo.
    """
    import torch
    import torch.distributed as dist

    from .records import estimate_moments_batch, seed_words

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    N = int(X.shape[0])
    lo, hi = shard_range(N, rank, world)
    idx = np.arange(lo, hi)
    seeds = seed_words(cfg_seed, 401, idx)
    if builder is None:
        Xs = torch.as_tensor(np.asarray(X)[lo:hi], device="cuda")
        S = torch.as_tensor(seeds.astype(np.int32), device="cuda")
        res = estimate_moments_batch(scene, Xs, seeds=S, epsilon=kw.pop("epsilon", 0.05), **kw)
        local = res.records
    else:
        local = builder(scene, np.asarray(X)[lo:hi], seeds)
    return all_gather_rows(local, group=group), (lo, hi)
