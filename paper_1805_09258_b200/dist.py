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


def broadcast_cache_set(cache_set, src: int = 0, group=None):
    """Make every rank's CacheSet hold `src`'s records, in `src`'s insertion order.

    Used after a populate on one rank (the reference's sequential insertion order is
    what the lookup sums follow) before a sharded frozen render.  Records travel as
    packed float64 rows (position, value, grad, axes, radii): counts first, then rows.
    Under NCCL the rows never leave the device: `src` reads them out of its device cache
    (vc_cache_records), the broadcast runs over NVLink, and receivers append them to an
    emptied device cache (vc_cache_insert) — no host record objects on either side.
    """
    import torch
    import torch.distributed as dist

    from .records import record_size

    dev = _coll_device(group)
    on_gpu = dev.type == "cuda"
    me = dist.get_rank(group)
    for cache in (cache_set.single, cache_set.multiple):
        rows = None
        if me == src:
            rows = cache.device_rows() if on_gpu else torch.from_numpy(cache.packed())
        n = torch.tensor([0 if rows is None else rows.shape[0]], dtype=torch.int64, device=dev)
        dist.broadcast(n, src, group=group)
        k = int(n.item())
        buf = rows if rows is not None else torch.zeros((k, record_size(cache.dim)), dtype=torch.float64, device=dev)
        if k:
            dist.broadcast(buf, src, group=group)
        if me != src:
            cache.clear()
            if on_gpu:
                torch.cuda.synchronize()
                cache.insert_device_rows(buf, k)
            else:
                cache.extend_packed(buf.numpy())
    return cache_set


def render_sharded(scene, camera, settings, cache_set, *, renderer=None, group=None):
    """Frozen-cache camera render with image rows sharded over ranks.

    Every rank holds the same cache set (e.g. via `broadcast_cache_set`); rank r marches
    rows shard_range(height, r, world), and the row slabs are all-gathered into the full
    image (height × width × 3 float64) on every rank.  Per-pixel RNG streams depend only
    on the global pixel index (seeds (seed, 211, k, i, m), src/renderer.py:471), so the
    image equals the single-process render whatever the sharding.  Returns (image, stats)
    with cache_hits / direct_evaluations summed over ranks.
    `renderer(scene, camera, settings, cache_set, row0, rows) -> (slab, stats)` defaults to
    the device march (`renderer.render_rows`); tests substitute a CPU stand-in.
    """
    import torch
    import torch.distributed as dist

    from . import renderer as R

    if not settings.frozen and settings.mode != "path":
        raise ValueError("render_sharded requires frozen=True (insertion order is sequential)")
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    lo, hi = shard_range(int(camera.height), rank, world)
    fn = renderer if renderer is not None else R.render_rows
    slab, st = fn(scene, camera, settings, cache_set, lo, hi - lo)
    dev = _coll_device(group)
    full = all_gather_rows(torch.as_tensor(np.ascontiguousarray(slab), dtype=torch.float64).to(dev), group=group)
    cnt = torch.tensor([st["cache_hits"], st["direct_evaluations"]], dtype=torch.int64, device=dev)
    if settings.mode == "path":  # render() reports no cache statistics in path mode (src/renderer.py:409-421)
        cnt.zero_()
    dist.all_reduce(cnt, group=group)
    image = full.cpu().numpy().reshape(int(camera.height), int(camera.width), 3)
    return image, {"cache_hits": int(cnt[0]), "direct_evaluations": int(cnt[1]), "rows": (lo, hi)}


def _coll_device(group=None):
    """Tensors for a collective live on the current GPU under NCCL, on the CPU under gloo."""
    import torch
    import torch.distributed as dist

    if dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")
