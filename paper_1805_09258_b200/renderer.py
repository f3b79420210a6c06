"""Render orchestration on the B200 path: settings, targets, CacheSet, populate_cache, render.

Mirrors src/renderer.py:45-131 (RenderSettings, FieldGrid), :134-193 (Camera),
:201-275 (CacheSet), :282-327 (populate_cache) and :402-484 (render) for the cache
modes "ours-aniso" / "ours-iso" — same names, argument meaning, return values and
ValueError / TypeError cases.  The march, the sequential-exact cache population and
every record build, lookup and image accumulation run in libvolcache_b200.so
(vc_populate, vc_render_field, vc_render); this module only validates and packs.

The occlusion-unaware "baseline" mode runs on the device too (vc_baseline_records,
log-space blend), and so does the path-traced reference mode "path" (vc_path_trace).
Out of scope: the deterministic "quadrature" oracle mode, which raises
NotImplementedError.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .baseline import baseline_estimate, log_space_interpolate, make_baseline_record
from .cache import RadianceCache, interpolate
from .records import DEFAULT_N_ANGULAR, device_scene, estimate_moments, make_record

MODES = ("ours-aniso", "ours-iso", "baseline", "path", "quadrature")
CACHE_MODES = ("ours-aniso", "ours-iso", "baseline")
DEVICE_MODES = ("ours-aniso", "ours-iso", "baseline")


def _unsupported(mode: str):
    return NotImplementedError(
        f"mode {mode!r} is outside the B200 hot path (DESIGN.md §6); use the reference for it")


@dataclass(frozen=True)
class RenderSettings:
    """Knobs shared by populate/render (src/renderer.py:50-85)."""

    mode: str = "ours-aniso"
    epsilon: float = 0.05
    spp: int = 16
    march_step: float = 0.1
    n_angular: int | None = None
    seed: int = 0
    frozen: bool = True
    max_media_bounces: int = 2
    n_light_samples: int = 16
    n_inner: int = 1
    baseline_alpha: float = 1.0
    path_samples_per_point: int = 256
    quad_gather_grid: int = 96
    quad_n_secondary: int = 256
    quad_n_angular: int = 512
    quad_n_dist: int = 24
    quad3d_n_angular: int = 256
    quad3d_n_dist: int = 12
    quad3d_n_secondary: int = 64

    def __post_init__(self):
        if self.mode not in MODES:
            raise ValueError(f"mode must be one of {MODES}, got {self.mode!r}")
        if self.epsilon <= 0.0:
            raise ValueError("epsilon must be positive")
        if self.march_step <= 0.0:
            raise ValueError("march_step must be positive")
        if self.spp < 1:
            raise ValueError("spp must be at least 1")


@dataclass(frozen=True)
class FieldGrid:
    """2D cell-center evaluation grid in display orientation, row 0 = top (src/renderer.py:88-131)."""

    bounds_min: np.ndarray
    bounds_max: np.ndarray
    nx: int
    ny: int

    def __post_init__(self):
        object.__setattr__(self, "bounds_min", np.asarray(self.bounds_min, dtype=float))
        object.__setattr__(self, "bounds_max", np.asarray(self.bounds_max, dtype=float))
        if self.bounds_min.shape != (2,) or self.bounds_max.shape != (2,):
            raise ValueError("FieldGrid bounds must be 2-vectors")
        if np.any(self.bounds_max <= self.bounds_min):
            raise ValueError("FieldGrid bounds must have positive extent")
        if self.nx < 1 or self.ny < 1:
            raise ValueError("FieldGrid resolution must be positive")

    @classmethod
    def for_scene(cls, scene, nx: int, ny: int) -> "FieldGrid":
        if scene.dim != 2:
            raise ValueError("FieldGrid targets require a 2D scene")
        return cls(scene.bounds_min, scene.bounds_max, nx, ny)

    def cell_center(self, iy: int, ix: int) -> np.ndarray:
        dx = (self.bounds_max[0] - self.bounds_min[0]) / self.nx
        dy = (self.bounds_max[1] - self.bounds_min[1]) / self.ny
        return np.array([self.bounds_min[0] + (ix + 0.5) * dx, self.bounds_max[1] - (iy + 0.5) * dy])

    @property
    def centers(self) -> np.ndarray:
        dx = (self.bounds_max[0] - self.bounds_min[0]) / self.nx
        dy = (self.bounds_max[1] - self.bounds_min[1]) / self.ny
        xs = self.bounds_min[0] + (np.arange(self.nx) + 0.5) * dx
        ys = self.bounds_max[1] - (np.arange(self.ny) + 0.5) * dy
        gx, gy = np.meshgrid(xs, ys)
        return np.stack([gx, gy], axis=-1)


@dataclass(frozen=True)
class Camera:
    """Pinhole camera for 3D scenes; fov_degrees is the vertical field of view (src/renderer.py:134-170)."""

    position: np.ndarray
    look_at: np.ndarray
    up: np.ndarray
    fov_degrees: float
    width: int
    height: int

    def __post_init__(self):
        vals = {}
        for name in ("position", "look_at", "up"):
            v = np.asarray(getattr(self, name), dtype=float)
            if v.shape != (3,):
                raise ValueError(f"camera {name} must be a 3-vector")
            vals[name] = v
            object.__setattr__(self, name, v)
        if not 0.0 < self.fov_degrees < 180.0:
            raise ValueError("fov_degrees must lie in (0, 180)")
        if self.width < 1 or self.height < 1:
            raise ValueError("camera resolution must be positive")
        forward = vals["look_at"] - vals["position"]
        if np.linalg.norm(forward) == 0.0:
            raise ValueError("camera look_at must differ from position")
        if np.linalg.norm(np.cross(forward / np.linalg.norm(forward), vals["up"])) < 1e-9:
            raise ValueError("camera up must not be parallel to the view direction")

    def _c(self) -> "_lib.Camera":
        cam = _lib.Camera()
        cam.position[:] = [float(v) for v in self.position]
        cam.look_at[:] = [float(v) for v in self.look_at]
        cam.up[:] = [float(v) for v in self.up]
        cam.fov_degrees = float(self.fov_degrees)
        cam.width = int(self.width)
        cam.height = int(self.height)
        return cam


def _seed(*parts) -> np.random.SeedSequence:
    """SeedSequence of 32-bit-masked parts (src/renderer.py:278-279)."""
    return np.random.SeedSequence([int(p) & 0xFFFFFFFF for p in parts])


def _check_target(scene, target) -> None:
    """src/renderer.py:371-379."""
    if isinstance(target, FieldGrid):
        if scene.dim != 2:
            raise ValueError("FieldGrid rendering requires a 2D scene")
    elif isinstance(target, Camera):
        if scene.dim != 3:
            raise ValueError("Camera rendering requires a 3D scene")
    else:
        raise TypeError("target must be a FieldGrid or a Camera")


def _n_angular(scene, settings) -> int:
    return int(settings.n_angular if settings.n_angular is not None else DEFAULT_N_ANGULAR[scene.dim])


def _params(scene, target, settings) -> "_lib.PopulateParams":
    p = _lib.PopulateParams()
    if isinstance(target, FieldGrid):
        p.target = _lib.VC_TARGET_FIELD
        p.field_nx, p.field_ny = int(target.nx), int(target.ny)
        p.field_min[:] = [float(v) for v in target.bounds_min]
        p.field_max[:] = [float(v) for v in target.bounds_max]
    else:
        p.target = _lib.VC_TARGET_CAMERA
        p.camera = target._c()
    p.march_step = float(settings.march_step)
    p.seed = int(settings.seed) & 0xFFFFFFFF  # _seed masks every part to 32 bits (src/renderer.py:278-279)
    p.n_angular = _n_angular(scene, settings)
    p.n_inner = int(settings.n_inner)
    p.n_light_samples = int(settings.n_light_samples)
    p.epsilon = float(settings.epsilon)
    p.isotropic = 1 if settings.mode == "ours-iso" else 0
    p.estimator = _estimator(settings.mode)
    p.max_media_bounces = int(settings.max_media_bounces)
    p.baseline_alpha = float(settings.baseline_alpha)
    p.path_samples = int(settings.path_samples_per_point)
    return p


def _estimator(mode: str) -> int:
    return {"baseline": _lib.VC_EST_BASELINE, "path": _lib.VC_EST_PATH}.get(mode, _lib.VC_EST_SUBDIVISION)


class CacheSet:
    """Paired single/multiple-scattering caches built by one estimator mode (src/renderer.py:201-275)."""

    def __init__(self, scene, mode: str, *, _single=None, _multiple=None):
        if mode not in CACHE_MODES:
            raise ValueError(f"cache modes are {CACHE_MODES}, got {mode!r}")
        if mode not in DEVICE_MODES:
            raise _unsupported(mode)
        self.mode = mode
        self.scene = scene
        self.single = _single if _single is not None else RadianceCache(scene.bounds_min, scene.bounds_max)
        self.multiple = _multiple if _multiple is not None else RadianceCache(scene.bounds_min, scene.bounds_max)

    @property
    def record_count(self) -> int:
        return len(self.single) + len(self.multiple)

    def lookup_parts(self, x):
        if self.mode == "baseline":
            return log_space_interpolate(self.single, x), log_space_interpolate(self.multiple, x)
        return interpolate(self.single, x), interpolate(self.multiple, x)

    def _handles(self):
        """Device caches flagged with this mode's blend (log-space for baseline)."""
        log = 1 if self.mode == "baseline" else 0
        hs, hm = self.single.handle(), self.multiple.handle()
        _lib.check(_lib.lib().vc_cache_set_blend(hs, log))
        _lib.check(_lib.lib().vc_cache_set_blend(hm, log))
        return hs, hm

    def lookup(self, x):
        s, m = self.lookup_parts(x)
        if s is None or m is None:
            return None
        return s + m

    def compute(self, x, settings: RenderSettings, rng_seed):
        """Fresh estimates at x → (total J, (record_single, record_multiple))."""
        scene = self.scene
        if self.mode == "baseline":
            est_s, est_m = baseline_estimate(scene, x, n_angular=settings.n_angular, rng_seed=rng_seed,
                                             max_media_bounces=settings.max_media_bounces,
                                             n_light_samples=settings.n_light_samples)
            rec_s = make_baseline_record(x, est_s, scene.scale, settings.baseline_alpha)
            rec_m = make_baseline_record(x, est_m, scene.scale, settings.baseline_alpha)
            return est_s.value + est_m.value, (rec_s, rec_m)
        mom_s, mom_m = estimate_moments(scene, x, n_angular=settings.n_angular, march_step=settings.march_step,
                                        rng_seed=rng_seed, n_inner=settings.n_inner,
                                        n_light_samples=settings.n_light_samples)
        aniso = self.mode == "ours-aniso"
        rec_s = make_record(x, mom_s, settings.epsilon, scene.scale, scene.max_emission, anisotropic=aniso)
        rec_m = make_record(x, mom_m, settings.epsilon, scene.scale, scene.max_emission, anisotropic=aniso)
        return mom_s.L + mom_m.L, (rec_s, rec_m)

    def insert(self, records, which=(True, True)) -> None:
        rec_s, rec_m = records
        if which[0]:
            self.single.insert(rec_s)
        if which[1]:
            self.multiple.insert(rec_m)


def populate_cache(scene, target, settings: RenderSettings, *, window: int = 0, lookahead: int = 0,
                   build_hook=None):
    """March view points in scanline order, inserting records where coverage lacks.

    Returns (CacheSet, stats) equal to the reference's sequential loop
    (src/renderer.py:302-327), computed by the speculative-window engine (vc_populate).
    `window` / `lookahead` bound the speculative builds per window and the initial
    lookahead (0 = library defaults); the result does not depend on them.
    `build_hook(n, x_ptr, words_ptr, seed_words, rec_ptr, stats_ptr) -> None` (device
    pointers) replaces the engine's record build for every speculative wave — the
    multi-GPU populate (`dist.populate_sharded`) shards each wave over ranks there.
    """
    if settings.mode not in CACHE_MODES:
        raise ValueError(f"populate_cache requires a cache mode, got {settings.mode!r}")
    _check_target(scene, target)
    if settings.mode not in DEVICE_MODES:
        raise _unsupported(settings.mode)
    start = time.perf_counter()
    ds = device_scene(scene)
    p = _params(scene, target, settings)
    p.window = int(window)
    p.lookahead = int(lookahead)
    failure = []
    if build_hook is not None:
        if settings.mode not in ("ours-aniso", "ours-iso"):
            raise ValueError("build_hook applies to the subdivision estimator (modes ours-aniso / ours-iso)")

        def _hook(user, n, x, words, seed_words, rec, stats, stream):
            try:
                build_hook(int(n), int(x or 0), int(words or 0), int(seed_words), int(rec or 0), int(stats or 0))
                return 0
            except BaseException as exc:  # reported after vc_populate returns
                failure.append(exc)
                return 1

        cb = _lib.BUILD_HOOK(_hook)
        p.build_hook = _lib.C.cast(cb, _lib.C.c_void_p)
    hs, hm = _lib.C.c_void_p(), _lib.C.c_void_p()
    st = np.zeros(8, np.int64)
    rc = _lib.lib().vc_populate(ds.handle, _lib.C.byref(p), _lib.C.byref(hs), _lib.C.byref(hm), _lib.ptr(st), None)
    if failure:
        raise failure[0]
    _lib.check(rc)
    single = RadianceCache._adopt(scene.bounds_min, scene.bounds_max, hs)
    multiple = RadianceCache._adopt(scene.bounds_min, scene.bounds_max, hm)
    single.sphere_records = multiple.sphere_records = settings.mode == "baseline"
    cs = CacheSet(scene, settings.mode, _single=single, _multiple=multiple)
    stats = {
        "mode": settings.mode,
        "points_marched": int(st[0]),
        "records": int(st[1] + st[2]),
        "records_single": int(st[1]),
        "records_multiple": int(st[2]),
        "seconds": time.perf_counter() - start,
        "windows": int(st[3]),
        "builds": int(st[4]),
        "discarded_builds": int(st[5]),
        "early_stops": int(st[6]),
    }
    return cs, stats


def _render_params(scene, settings: RenderSettings) -> "_lib.RenderParams":
    rp = _lib.RenderParams()
    rp.spp = int(settings.spp)
    rp.march_step = float(settings.march_step)
    rp.seed = int(settings.seed) & 0xFFFFFFFF
    rp.n_angular = _n_angular(scene, settings)
    rp.n_inner = int(settings.n_inner)
    rp.n_light_samples = int(settings.n_light_samples)
    rp.epsilon = float(settings.epsilon)
    rp.estimator = _estimator(settings.mode)
    rp.max_media_bounces = int(settings.max_media_bounces)
    rp.path_samples = int(settings.path_samples_per_point)
    rp.grow = 0 if settings.frozen else 1
    rp.isotropic = 1 if settings.mode == "ours-iso" else 0
    rp.baseline_alpha = float(settings.baseline_alpha)
    return rp


def render_rows(scene, camera: Camera, settings: RenderSettings, cache_set: CacheSet, row0: int, rows: int):
    """Frozen camera render of image rows [row0, row0 + rows) → (slab (rows, width, 3), stats).

    The rows equal the same rows of `render(scene, camera, settings, cache_set)`: every
    pixel's streams depend on its global index (src/renderer.py:440-484).  The unit of the
    row-sharded multi-GPU render (`dist.render_sharded`).
    """
    _check_target(scene, camera)
    if not isinstance(camera, Camera):
        raise TypeError("render_rows takes a Camera target")
    if settings.mode not in DEVICE_MODES + ("path",):
        raise _unsupported(settings.mode)
    if settings.mode == "path":  # every point path-traced, as render() (src/renderer.py:337-346)
        settings = RenderSettings(**{**settings.__dict__, "frozen": True})
    if not settings.frozen:
        raise ValueError("render_rows requires frozen=True")
    if not 0 <= row0 <= row0 + rows <= camera.height:
        raise ValueError("row range outside the image")
    if settings.mode == "path":
        cache_set = CacheSet(scene, "ours-aniso")
    image = np.zeros((camera.height, camera.width, 3))
    out = np.zeros(2, np.int64)
    if rows > 0:
        cam = camera._c()
        cam.row0, cam.rows, cam.col0, cam.cols = int(row0), int(rows), 0, int(camera.width)
        rp = _render_params(scene, settings)
        hs, hm = cache_set._handles()
        _lib.check(_lib.lib().vc_render(device_scene(scene).handle, hs, hm, _lib.C.byref(cam), _lib.C.byref(rp),
                                        _lib.ptr(image), _lib.ptr(out), _lib.VC_MEM_HOST, None))
    if settings.mode == "path":  # path mode keeps no cache statistics (src/renderer.py:337-346)
        out[:] = 0
    return image[row0:row0 + rows].copy(), {"cache_hits": int(out[0]), "direct_evaluations": int(out[1])}


def render(scene, target, settings: RenderSettings, cache_set: CacheSet = None):
    """Render the target; returns (image, stats) (src/renderer.py:402-422).

    Cache modes populate a fresh cache first unless one is passed in.  Field images hold
    the in-scatter source density; camera images hold radiance.
    """
    _check_target(scene, target)
    if settings.mode not in DEVICE_MODES + ("path",):
        raise _unsupported(settings.mode)
    start = time.perf_counter()
    stats = {"mode": settings.mode, "cache_hits": 0, "direct_evaluations": 0}
    path = settings.mode == "path"
    if path:  # every shading point path-traced: an empty cache pair, frozen (src/renderer.py:337-346)
        cache_set = CacheSet(scene, "ours-aniso")
        settings = RenderSettings(**{**settings.__dict__, "frozen": True})
    elif cache_set is None:
        cache_set, pop_stats = populate_cache(scene, target, settings)
        stats["populate"] = pop_stats
    if not path:
        stats["records"] = cache_set.record_count
    ds = device_scene(scene)
    out = np.zeros(2, np.int64)
    if isinstance(target, FieldGrid):
        p = _params(scene, target, settings)
        image = np.zeros((target.ny, target.nx, 3))
        hs, hm = cache_set._handles()
        _lib.check(_lib.lib().vc_render_field(ds.handle, hs, hm, _lib.C.byref(p), 1 if settings.frozen else 0,
                                              _lib.ptr(image), _lib.ptr(out), _lib.VC_MEM_HOST, None))
        if not settings.frozen:
            cache_set.single._device_changed()
            cache_set.multiple._device_changed()
    else:
        cam = target._c()
        rp = _render_params(scene, settings)
        image = np.zeros((target.height, target.width, 3))
        hs, hm = cache_set._handles()
        _lib.check(_lib.lib().vc_render(ds.handle, hs, hm, _lib.C.byref(cam), _lib.C.byref(rp), _lib.ptr(image),
                                        _lib.ptr(out), _lib.VC_MEM_HOST, None))
        if not settings.frozen:
            cache_set.single._device_changed()
            cache_set.multiple._device_changed()
    if not path:  # the reference counts hits/evaluations only in the cache modes
        stats["cache_hits"] = int(out[0])
        stats["direct_evaluations"] = int(out[1])
    if not settings.frozen:
        stats["records"] = cache_set.record_count
    stats["seconds"] = time.perf_counter() - start
    return image, stats
