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


def sharded_wave(n: int, build_local, exchange, rank: int, world: int):
    """One speculative build wave of n points split over ranks: rank r builds its contiguous
    share [lo, hi) (`build_local(lo, hi)` → (hi − lo, K) rows) and `exchange` all-gathers the
    shares into the (n, K) rows in wave order.  Every record's seed words come with its point,
    so the rows equal a single-rank build of the whole wave."""
    lo, hi = shard_range(n, rank, world)
    return exchange(build_local(lo, hi))


class _DeviceArray:
    """Zero-copy CUDA array view of a raw device pointer (__cuda_array_interface__)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(int(v) for v in shape), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3, "strides": None}


def _view(ptr: int, shape, dtype):
    import torch

    typestr = {torch.float64: "<f8", torch.int64: "<i8", torch.int32: "<i4"}[dtype]
    if ptr == 0 or 0 in tuple(shape):
        return torch.empty(shape, dtype=dtype, device="cuda")
    return torch.as_tensor(_DeviceArray(ptr, shape, typestr), device="cuda")


def populate_sharded(scene, target, settings, *, group=None, window: int = 0, lookahead: int = 0):
    """populate_cache (src/renderer.py:302-327) on every rank of the group, with each
    speculative build wave of the engine sharded over the ranks.

    Every rank runs the same deterministic engine (march stream, cover tests, sequential
    resolve); only the record builds are split: rank r builds its contiguous share of each
    wave and the shares are all-gathered device-to-device over NCCL before the resolve, so
    every rank commits the same records in the same order — the caches equal the
    single-GPU (and the reference's sequential) populate record for record.
    Returns (CacheSet, stats) on every rank.
    """
    import torch
    import torch.distributed as dist

    from . import _lib
    from . import renderer as R
    from .records import device_scene, record_size

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    ds = device_scene(scene)
    d = ds.dim
    RS = record_size(d)
    prm = _lib.BuildParams()
    prm.n_angular = R._n_angular(scene, settings)
    prm.march_step = float(settings.march_step)
    prm.n_inner = int(settings.n_inner)
    prm.n_light_samples = int(settings.n_light_samples)
    prm.epsilon = float(settings.epsilon)
    prm.flags = _lib.VC_SEED_WORDS | _lib.VC_MAKE_RECORDS | (_lib.VC_ISOTROPIC if settings.mode == "ours-iso" else 0)
    L = _lib.lib()

    def hook(n, x, w, sw, rec, stats):
        prm.seed_words = sw
        X = _view(x, (n, d), torch.float64)
        Wd = _view(w, (n, sw), torch.int32)

        def build_local(lo, hi):
            m = hi - lo
            recs = torch.zeros((m, 2 * RS), dtype=torch.float64, device="cuda")
            st = torch.zeros((m, 8), dtype=torch.int64, device="cuda")
            if m:
                xs, ws = X[lo:hi].contiguous(), Wd[lo:hi].contiguous()
                _lib.check(L.vc_build_records(ds.handle, m, _lib.C.c_void_p(xs.data_ptr()),
                                              _lib.C.c_void_p(ws.data_ptr()), None, _lib.C.byref(prm), None,
                                              _lib.C.c_void_p(st.data_ptr()), _lib.C.c_void_p(recs.data_ptr()),
                                              None))
            return torch.cat([recs, st.view(torch.float64)], dim=1)

        rows = sharded_wave(n, build_local, lambda t: all_gather_rows(t, group=group), rank, world)
        _view(rec, (n, 2 * RS), torch.float64).copy_(rows[:, :2 * RS])
        _view(stats, (n, 8), torch.int64).copy_(rows[:, 2 * RS:].contiguous().view(torch.int64))

    return R.populate_cache(scene, target, settings, window=window, lookahead=lookahead, build_hook=hook)


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
