"""Record build drop-ins: estimate_moments / make_record on the B200 path.

Mirrors the reference interface (src/subdivision.py:111-128, :373-393;
src/cache.py:94-121, :153-189): same names, argument meaning, return types and
ValueError cases.  All arithmetic runs in libvolcache_b200.so; this module only
packs arguments.  A batch entry point (`estimate_moments_batch`) replaces the
reference's one-call-per-point Python loop.
"""

from __future__ import annotations

import weakref
from dataclasses import dataclass

import numpy as np

from . import _lib
from .scene import scene_arrays

DEFAULT_N_ANGULAR = {2: 256, 3: 16384}  # src/subdivision.py:49


def moment_size(d: int) -> int:
    return 3 + 3 * d + 3 * d * d


def record_size(d: int) -> int:
    return d + 3 + 3 * d + d * d + d


@dataclass(frozen=True)
class Moments:
    """Radiance value, gradient and Hessian per channel (src/subdivision.py:111-122)."""

    L: np.ndarray
    grad: np.ndarray
    hess: np.ndarray
    kind: str

    @property
    def dim(self) -> int:
        return self.grad.shape[1]


# Result class of estimate_moments: a host that rebinds the reference's names can have the
# drop-in return the reference's own Moments dataclass (same fields), so isinstance checks
# on the reference side hold (tools/rebind_plugin.py).
_RESULT_TYPES = {"moments": Moments}


def use_result_types(moments=None) -> None:
    """Return `moments(L=, grad=, hess=, kind=)` instances from estimate_moments (None: ours)."""
    _RESULT_TYPES["moments"] = moments if moments is not None else Moments


@dataclass(frozen=True)
class CacheRecord:
    """Value + gradient with an ellipsoidal valid region (src/cache.py:94-121)."""

    position: np.ndarray
    value: np.ndarray
    grad: np.ndarray
    axes: np.ndarray
    radii: np.ndarray

    @property
    def dim(self) -> int:
        return self.position.size

    @property
    def bounding_radius(self) -> float:
        return float(np.max(self.radii))

    def pack(self) -> np.ndarray:
        return np.concatenate([self.position, self.value, self.grad.ravel(), self.axes.ravel(), self.radii])


@dataclass(frozen=True)
class BaselineRecord:
    """Sphere record of the occlusion-unaware baseline (src/cache.py:124-145).

    The device stores it like an ellipse record: identity axes, every radius = `radius`.
    """

    position: np.ndarray
    value: np.ndarray
    grad: np.ndarray
    radius: float

    @property
    def dim(self) -> int:
        return self.position.size

    @property
    def bounding_radius(self) -> float:
        return self.radius

    @property
    def axes(self) -> np.ndarray:
        return np.eye(self.dim)

    @property
    def radii(self) -> np.ndarray:
        return np.full(self.dim, float(self.radius))


def unpack_record(row, d: int) -> CacheRecord:
    row = np.asarray(row, float)
    o = 0

    def take(k):
        nonlocal o
        v = row[o:o + k].copy()
        o += k
        return v

    pos = take(d)
    val = take(3)
    grad = take(3 * d).reshape(3, d)
    axes = take(d * d).reshape(d, d)
    radii = take(d)
    return CacheRecord(pos, val, grad, axes, radii)


class DeviceScene:
    """A scene uploaded to the current CUDA device (BVH built once, src/scene.py:124-219)."""

    def __init__(self, scene):
        dim, V, E, A = scene_arrays(scene)
        self.dim = dim
        self.bounds_min = np.ascontiguousarray(np.asarray(scene.bounds_min, float))
        self.bounds_max = np.ascontiguousarray(np.asarray(scene.bounds_max, float))
        self.sigma_s = float(scene.medium.sigma_s)
        self.sigma_a = float(scene.medium.sigma_a)
        self.scale = float(np.linalg.norm(self.bounds_max - self.bounds_min))
        self.max_emission = float(E.max()) if E.size else 0.0
        self.n_surfaces = V.shape[0]
        h = _lib.C.c_void_p()
        L = _lib.lib()
        _lib.check(L.vc_scene_create(dim, V.shape[0], _lib.ptr(V), _lib.ptr(E), _lib.ptr(A),
                                     _lib.ptr(self.bounds_min), _lib.ptr(self.bounds_max),
                                     self.sigma_s, self.sigma_a, _lib.C.byref(h)))
        self.handle = h
        self._finalizer = weakref.finalize(self, L.vc_scene_destroy, h)
        lights = getattr(scene, "lights", None)  # extension: delta lights (scene.light_rows)
        if lights is not None and len(lights):
            rows = np.ascontiguousarray(np.asarray(lights, float).reshape(-1, 8))
            _lib.check(L.vc_scene_set_lights(h, rows.shape[0], _lib.ptr(rows)))

    def set_budget(self, nbytes: int) -> None:
        _lib.check(_lib.lib().vc_scene_set_budget(self.handle, int(nbytes)))

    def contains(self, pts) -> np.ndarray:
        pts = np.atleast_2d(np.asarray(pts, float))
        eps = 1e-12 * self.scale
        return np.all((pts >= self.bounds_min - eps) & (pts <= self.bounds_max + eps), axis=1)


_SCENES: dict[int, tuple] = {}


def device_scene(scene) -> DeviceScene:
    """Upload `scene` once per object (cached by identity while the object lives)."""
    if isinstance(scene, DeviceScene):
        return scene
    key = id(scene)
    hit = _SCENES.get(key)
    if hit is not None and hit[0]() is scene:
        return hit[1]
    ds = DeviceScene(scene)
    try:
        ref = weakref.ref(scene, lambda _r, k=key: _SCENES.pop(k, None))
    except TypeError:  # not weak-referenceable: keep it alive with the handle
        ref = (lambda s=scene: s)
    _SCENES[key] = (ref, ds)
    return ds


def pcg64_state(rng_seed) -> tuple[np.ndarray, np.random.Generator]:
    """numpy default_rng(rng_seed) PCG64 state as (state_hi, state_lo, inc_hi, inc_lo)."""
    g = np.random.default_rng(rng_seed)
    st = g.bit_generator.state
    if st.get("bit_generator") != "PCG64":
        raise ValueError("only PCG64 generators (numpy default_rng) are supported")
    s, inc = int(st["state"]["state"]), int(st["state"]["inc"])
    m = (1 << 64) - 1
    return np.array([s >> 64, s & m, inc >> 64, inc & m], dtype=np.uint64), g


def _params(dim, n_angular, march_step, n_inner, n_light_samples, epsilon, flags, seed_words=0, media_bounces=1,
            hg_g=0.0):
    p = _lib.BuildParams()
    p.media_bounces = int(media_bounces)
    p.hg_g = float(hg_g)
    p.n_angular = int(DEFAULT_N_ANGULAR[dim] if n_angular is None else n_angular)
    p.march_step = float(march_step)
    p.n_inner = int(n_inner)
    p.n_light_samples = int(n_light_samples)
    p.epsilon = float(epsilon) if epsilon is not None else 0.05
    p.flags = int(flags)
    p.seed_words = int(seed_words)
    return p


def _draws(dim, n, P, n_inner, media_bounces=1):
    per = 1 if dim == 2 else 2
    return per * n + P * n_inner * per + P * n_inner * max(0, media_bounces - 1) * (per + 1)


def estimate_moments(scene, x, n_angular=None, march_step=0.1, rng_seed=None, n_inner=1,
                     n_light_samples=16, adjacency=None, media_bounces=1, hg_g=0.0):
    """(single, multiple) Moments at x — drop-in for src/subdivision.py:373-393.

    `adjacency` optionally injects the 3D triangle list (e.g. qhull's simplices) instead
    of the GPU spherical Delaunay.  A Generator passed as rng_seed is advanced by the
    draws the build consumed, exactly as the reference would.  `media_bounces` > 1 is an
    extension (not in the reference): each media sample's gather path continues through up
    to media_bounces − 1 further media scattering events, and `hg_g` ≠ 0 makes those media
    scattering events Henyey–Greenstein.
    """
    ds = device_scene(scene)
    x = np.ascontiguousarray(np.asarray(x, float).reshape(-1))
    if x.size != ds.dim:
        raise ValueError("x dimensionality does not match the scene")
    if march_step <= 0.0:
        raise ValueError("march_step must be positive")
    if not ds.contains(x)[0]:
        raise ValueError("subdivision center lies outside the medium bounds")
    st, gen = pcg64_state(rng_seed)
    p = _params(ds.dim, n_angular, march_step, n_inner, n_light_samples, None, _lib.VC_MEM_HOST,
                media_bounces=media_bounces, hg_g=hg_g)
    d = ds.dim
    mom = np.zeros((2, moment_size(d)))
    stats = np.zeros(8, np.int64)
    adj = None
    if adjacency is not None and d == 3:
        adj = np.ascontiguousarray(np.asarray(adjacency, np.int32))
    _lib.check(_lib.lib().vc_build_records(ds.handle, 1, _lib.ptr(x), _lib.ptr(st), _lib.ptr(adj),
                                           _lib.C.byref(p), _lib.ptr(mom), _lib.ptr(stats), None, None))
    if isinstance(rng_seed, np.random.Generator):
        gen.bit_generator.advance(_draws(d, p.n_angular, int(stats[3]), p.n_inner, media_bounces))
    out = []
    for k, kind in enumerate(("single", "multiple")):
        L, g, h = split_moments(mom[k], d)
        out.append(_RESULT_TYPES["moments"](L=L, grad=g, hess=h, kind=kind))
    return out[0], out[1]


def split_moments(row, d):
    row = np.asarray(row)
    L = row[:3].copy()
    g = row[3:3 + 3 * d].reshape(3, d).copy()
    h = row[3 + 3 * d:].reshape(3, d, d).copy()
    return L, g, h


@dataclass
class BatchResult:
    """Stacked batch outputs: moments (N, 2, M), stats (N, 8), records (N, 2, RS) or None."""

    dim: int
    moments: object
    stats: object
    records: object = None

    @property
    def L(self):
        return self.moments[:, :, :3]

    @property
    def grad(self):
        d = self.dim
        return self.moments[:, :, 3:3 + 3 * d].reshape(-1, 2, 3, d)

    @property
    def hess(self):
        d = self.dim
        return self.moments[:, :, 3 + 3 * d:].reshape(-1, 2, 3, d, d)


def estimate_moments_batch(scene, X, seeds=None, rng_states=None, n_angular=None, march_step=0.1,
                           n_inner=1, n_light_samples=16, adjacency=None, epsilon=None,
                           anisotropic=True, stream=None, media_bounces=1, hg_g=0.0,
                           defer_check=False) -> BatchResult:
    """Batch record build: N cache points in one call (moments, stats, optional records).

    X is (N, d) host numpy or a CUDA torch tensor (then every output is a CUDA tensor
    and the call is asynchronous on `stream`).  Per-record RNG: `seeds` (N, w) uint32
    SeedSequence entropy words — e.g. rows (cfg_seed, 401, i), src/renderer.py:317 —
    or `rng_states` (N, 4) uint64 PCG64 states.  `epsilon` set → also make_record.
    With CUDA inputs the reference's ValueError for a point outside the bounds needs one host
    read of a device flag per call; `defer_check=True` returns without it (successive calls
    then queue back to back) and `check_deferred()` raises for all of them at once.
    """
    ds = device_scene(scene)
    d = ds.dim
    on_dev = hasattr(X, "data_ptr") and getattr(X, "is_cuda", False)
    flags = 0 if on_dev else _lib.VC_MEM_HOST
    if seeds is not None:
        flags |= _lib.VC_SEED_WORDS
    if epsilon is not None:
        flags |= _lib.VC_MAKE_RECORDS
    if not anisotropic:
        flags |= _lib.VC_ISOTROPIC
    if on_dev and defer_check:
        flags |= _lib.VC_DEFER_CHECK
    N = int(X.shape[0])
    if N == 0:
        return BatchResult(d, np.zeros((0, 2, moment_size(d))), np.zeros((0, 8), np.int64),
                           np.zeros((0, 2, record_size(d))) if epsilon else None)
    if on_dev:
        import torch

        dev = X.device
        Xc = X.contiguous().to(torch.float64)
        rng = (seeds if seeds is not None else rng_states)
        if rng is None:
            raise ValueError("seeds or rng_states is required")
        rng = rng.contiguous()
        mom = torch.empty((N, 2, moment_size(d)), dtype=torch.float64, device=dev)
        stats = torch.empty((N, 8), dtype=torch.int64, device=dev)
        recs = torch.empty((N, 2, record_size(d)), dtype=torch.float64, device=dev) if epsilon else None
        adj = adjacency.contiguous().to(torch.int32) if (adjacency is not None and d == 3) else None
        if stream is None:
            stream = torch.cuda.current_stream(dev).cuda_stream
    else:
        Xc = np.ascontiguousarray(np.asarray(X, float).reshape(N, d))
        if not np.all(ds.contains(Xc)):
            raise ValueError("subdivision center lies outside the medium bounds")
        if seeds is not None:
            rng = np.ascontiguousarray(np.asarray(seeds, dtype=np.uint32).reshape(N, -1))
        elif rng_states is not None:
            rng = np.ascontiguousarray(np.asarray(rng_states, dtype=np.uint64).reshape(N, 4))
        else:
            raise ValueError("seeds or rng_states is required")
        mom = np.zeros((N, 2, moment_size(d)))
        stats = np.zeros((N, 8), np.int64)
        recs = np.zeros((N, 2, record_size(d))) if epsilon else None
        adj = np.ascontiguousarray(np.asarray(adjacency, np.int32)) if (adjacency is not None and d == 3) else None
    p = _params(d, n_angular, march_step, n_inner, n_light_samples, epsilon, flags,
                seed_words=(rng.shape[1] if seeds is not None else 0), media_bounces=media_bounces, hg_g=hg_g)
    _lib.check(_lib.lib().vc_build_records(ds.handle, N, _lib.ptr(Xc), _lib.ptr(rng), _lib.ptr(adj),
                                           _lib.C.byref(p), _lib.ptr(mom), _lib.ptr(stats), _lib.ptr(recs),
                                           stream))
    return BatchResult(d, mom, stats, recs)


def check_deferred(stream=None) -> None:
    """Raise the ValueError of every `defer_check=True` build since the last call whose points
    left the medium bounds (vc_check_deferred); synchronises the stream."""
    if stream is None:
        import torch

        stream = torch.cuda.current_stream().cuda_stream
    _lib.check(_lib.lib().vc_check_deferred(stream))


def inspect_record(scene, x, rng_seed=None, n_angular=None, march_step=0.1, n_inner=1,
                   n_light_samples=16, adjacency=None, media_cap=1 << 22, media_bounces=1, hg_g=0.0):
    """One record with its per-direction internals (dirs, s, idx, counts, triangles, media)."""
    ds = device_scene(scene)
    d = ds.dim
    x = np.ascontiguousarray(np.asarray(x, float).reshape(-1))
    st, _ = pcg64_state(rng_seed)
    p = _params(d, n_angular, march_step, n_inner, n_light_samples, None, _lib.VC_MEM_HOST,
                media_bounces=media_bounces, hg_g=hg_g)
    n = p.n_angular
    dirs = np.zeros((n, d))
    s = np.zeros(n)
    idx = np.zeros(n, np.int32)
    cnt = np.zeros(n, np.int32)
    tris = np.zeros((2 * n - 4, 3), np.int32) if d == 3 else None
    media = np.zeros((media_cap, 3), np.float32)
    P = np.zeros(1, np.int64)
    mom = np.zeros((2, moment_size(d)))
    stats = np.zeros(8, np.int64)
    adj = np.ascontiguousarray(np.asarray(adjacency, np.int32)) if (adjacency is not None and d == 3) else None
    _lib.check(_lib.lib().vc_build_inspect(ds.handle, _lib.ptr(x), _lib.ptr(st), _lib.ptr(adj), _lib.C.byref(p),
                                           _lib.ptr(dirs), _lib.ptr(s), _lib.ptr(idx), _lib.ptr(cnt),
                                           _lib.ptr(tris), _lib.ptr(media), media_cap, _lib.ptr(P),
                                           _lib.ptr(mom), _lib.ptr(stats)))
    return {
        "dirs": dirs, "s": s, "idx": idx.astype(np.int64), "counts": cnt, "tris": tris,
        "media": media[: int(P[0])], "P": int(P[0]), "moments": mom, "stats": stats,
    }


def surface_radiance_batch(scene, idx, points, dirs, n_light_samples=16):
    """Outgoing radiance at surface hits — drop-in for src/transport.py:240-254: emission
    (two-sided) + albedo · direct lighting (emitter quadrature, one shadow ray per sample);
    idx < 0 → 0.  Returns (m, 3) float64."""
    ds = device_scene(scene)
    d = ds.dim
    idx = np.ascontiguousarray(np.asarray(idx).reshape(-1), np.int32)
    m = idx.size
    pts = np.ascontiguousarray(np.asarray(points, float).reshape(m, d))
    drs = np.ascontiguousarray(np.asarray(dirs, float).reshape(m, d))
    out = np.zeros((m, 3))
    if m:
        _lib.check(_lib.lib().vc_surface_radiance(ds.handle, m, _lib.ptr(pts), _lib.ptr(drs), _lib.ptr(idx),
                                                  int(n_light_samples), _lib.ptr(out), _lib.VC_MEM_HOST, None))
    return out


def make_records(X, moments, epsilon, scene_scale, max_emission, anisotropic=True):
    """Batch make_record: X (N, d), moments (N, 2, M) → packed records (N, 2, RS)."""
    X = np.ascontiguousarray(np.asarray(X, float))
    N, d = X.shape
    mom = np.ascontiguousarray(np.asarray(moments, float).reshape(N, 2, moment_size(d)))
    out = np.zeros((N, 2, record_size(d)))
    flags = _lib.VC_MEM_HOST | (0 if anisotropic else _lib.VC_ISOTROPIC)
    if epsilon <= 0.0:
        raise ValueError("epsilon must be positive")
    _lib.check(_lib.lib().vc_make_records(N, d, _lib.ptr(X), _lib.ptr(mom), float(epsilon), float(scene_scale),
                                          float(max_emission), flags, _lib.ptr(out), None))
    return out


def make_record(x, moments, epsilon, scene_scale, max_emission, anisotropic=True) -> CacheRecord:
    """Drop-in for src/cache.py:153-189 (eigen + radii on the GPU)."""
    x = np.asarray(x, float).reshape(-1)
    d = x.size
    row = np.zeros((1, 2, moment_size(d)))
    row[0, 0, :3] = moments.L
    row[0, 0, 3:3 + 3 * d] = np.asarray(moments.grad).ravel()
    row[0, 0, 3 + 3 * d:] = np.asarray(moments.hess).ravel()
    rec = make_records(x[None], row, epsilon, scene_scale, max_emission, anisotropic)
    return unpack_record(rec[0, 0], d)


def trace(scene, origins, dirs, with_bounds=False):
    """Nearest hit per ray → (t, idx): trace / trace_or_bounds (src/scene.py:271-315)."""
    ds = device_scene(scene)
    o = np.ascontiguousarray(np.asarray(origins, float).reshape(-1, ds.dim))
    d = np.ascontiguousarray(np.asarray(dirs, float).reshape(-1, ds.dim))
    m = o.shape[0]
    t = np.zeros(m)
    idx = np.zeros(m, np.int32)
    flags = _lib.VC_MEM_HOST | (_lib.VC_TRACE_BOUNDS if with_bounds else 0)
    _lib.check(_lib.lib().vc_trace(ds.handle, m, _lib.ptr(o), _lib.ptr(d), _lib.ptr(t), _lib.ptr(idx), flags, None))
    return t, idx.astype(np.int64)


def seed_words(cfg_seed: int, purpose: int, idx) -> np.ndarray:
    """(cfg_seed, purpose, i) rows as uint32 entropy words (src/renderer.py:278-279)."""
    idx = np.asarray(idx, dtype=np.int64)
    out = np.empty((idx.size, 3), np.uint32)
    out[:, 0] = np.uint32(int(cfg_seed) & 0xFFFFFFFF)
    out[:, 1] = np.uint32(int(purpose) & 0xFFFFFFFF)
    out[:, 2] = (idx & 0xFFFFFFFF).astype(np.uint32)
    return out
