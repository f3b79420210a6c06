"""Record cache, lookup and frozen-cache camera march on the B200 path.

Mirrors src/cache.py:262-360 (RadianceCache, interpolate) and the frozen camera
render of src/renderer.py:402-484.  Records live on the device behind a
multi-level grid index whose covering set equals the reference tree query
(≡ linear scan); interpolation and the march run in libvolcache_b200.so.
"""

from __future__ import annotations

import weakref

import numpy as np

from . import _lib
from .records import CacheRecord, device_scene, record_size


def _pack(recs, d: int) -> np.ndarray:
    """Record objects → packed rows (N, d + 3 + 3d + d² + d)."""
    if not recs:
        return np.zeros((0, record_size(d)))
    return np.ascontiguousarray(np.stack([np.concatenate([
        np.asarray(r.position, float), np.asarray(r.value, float), np.asarray(r.grad, float).ravel(),
        np.asarray(r.axes, float).ravel(), np.asarray(r.radii, float)]) for r in recs]))


class RadianceCache:
    """Records + exact point-query index (src/cache.py:262-334).

    Inserts are appended to the device copy lazily: the next lookup uploads only the
    records inserted since the last one (vc_cache_insert) and re-indexes on the device,
    so the reference's one-insert-per-miss loop (src/renderer.py:313-318) stays O(new)
    on the host.
    """

    MAX_DEPTH = 16

    def __init__(self, bounds_min, bounds_max):
        bmin = np.asarray(bounds_min, dtype=float)
        bmax = np.asarray(bounds_max, dtype=float)
        if bmin.shape != bmax.shape or bmin.size not in (2, 3):
            raise ValueError("bounds must be matching 2- or 3-vectors")
        if np.any(bmax <= bmin):
            raise ValueError("bounds_max must exceed bounds_min")
        self.bounds_min = np.ascontiguousarray(bmin)
        self.bounds_max = np.ascontiguousarray(bmax)
        self.dim = bmin.size
        self._records: list | None = []  # host record objects (None: held on the device only)
        self._synced = 0                  # records [0, _synced) are in the device cache
        self._handle = None
        self._fin = None
        self.sphere_records = False  # device-only rows are BaselineRecord spheres (baseline mode)

    @classmethod
    def _adopt(cls, bounds_min, bounds_max, handle) -> "RadianceCache":
        """Wrap a device cache built by the library (vc_populate); records download lazily."""
        c = cls(bounds_min, bounds_max)
        c._records = None
        c._set_handle(handle)
        c._synced = int(_lib.lib().vc_cache_size(handle))
        return c

    def _set_handle(self, h) -> None:
        self._handle = h
        self._fin = weakref.finalize(self, _lib.lib().vc_cache_destroy, h)

    def _device_changed(self) -> None:
        """The device cache grew in place (render with frozen=False): re-read lazily."""
        self._records = None
        self._synced = int(_lib.lib().vc_cache_size(self._handle))

    def _host_records(self) -> list:
        if self._records is None:
            rows = self._device_rows()
            from .records import unpack_record

            self._records = [unpack_record(r, self.dim) for r in rows]
        return self._records

    def _device_rows(self) -> np.ndarray:
        L = _lib.lib()
        n = int(L.vc_cache_size(self._handle))
        rows = np.zeros((n, record_size(self.dim)))
        if n:
            _lib.check(L.vc_cache_records(self._handle, _lib.ptr(rows), None, _lib.VC_MEM_HOST, None))
        return rows

    def __len__(self) -> int:
        if self._records is None:
            return int(_lib.lib().vc_cache_size(self._handle))
        return len(self._records)

    @property
    def records(self) -> list:
        return list(self._host_records())

    def insert(self, record) -> None:
        if np.asarray(record.position).size != self.dim:
            raise ValueError("record dimensionality does not match the cache")
        self._host_records().append(record)

    def extend_packed(self, packed: np.ndarray) -> None:
        """Insert many records given as packed rows (N, d + 3 + 3d + d² + d)."""
        from .records import unpack_record

        recs = self._host_records()
        for row in np.asarray(packed, float).reshape(-1, record_size(self.dim)):
            recs.append(unpack_record(row, self.dim))

    def clear(self) -> None:
        """Drop every record (host and device)."""
        if self._fin is not None:
            self._fin()
        self._handle = None
        self._fin = None
        self._records = []
        self._synced = 0

    def device_rows(self):
        """Packed rows as a CUDA float64 tensor (n, row) read on the device (no host copy)."""
        import torch

        h = self.handle()
        n = int(_lib.lib().vc_cache_size(h))
        out = torch.empty((n, record_size(self.dim)), dtype=torch.float64, device="cuda")
        if n:
            torch.cuda.synchronize()
            _lib.check(_lib.lib().vc_cache_records(h, _lib.C.c_void_p(out.data_ptr()), None, 0, None))
        return out

    def insert_device_rows(self, rows, n: int) -> None:
        """Append n packed rows that already sit in device memory (pointer or CUDA tensor),
        e.g. records received over NCCL: no host round trip, host objects re-read lazily."""
        h = self.handle()
        ptr = rows.data_ptr() if hasattr(rows, "data_ptr") else int(rows)
        _lib.check(_lib.lib().vc_cache_insert(h, int(n), _lib.C.c_void_p(ptr), 0, None))
        self._records = None
        self._synced += int(n)

    def packed(self) -> np.ndarray:
        if self._records is None:
            return self._device_rows()
        return _pack(self._records, self.dim)

    def handle(self):
        L = _lib.lib()
        if self._handle is None:
            recs = self.packed()
            h = _lib.C.c_void_p()
            _lib.check(L.vc_cache_create(self.dim, _lib.ptr(self.bounds_min), _lib.ptr(self.bounds_max),
                                         len(recs), _lib.ptr(recs) if len(recs) else None, _lib.C.byref(h)))
            self._set_handle(h)
            self._synced = len(recs)
        elif self._records is not None and len(self._records) > self._synced:
            rows = _pack(self._records[self._synced:], self.dim)
            _lib.check(L.vc_cache_insert(self._handle, len(rows), _lib.ptr(rows), _lib.VC_MEM_HOST, None))
            self._synced = len(self._records)
        return self._handle

    def interpolate_many(self, X, log_space: bool = False):
        """(J (m, 3) with NaN rows where uncovered, covering-record counts (m,)).

        log_space=True blends like log_space_interpolate (sphere records, src/cache.py:363-394).
        """
        X = np.ascontiguousarray(np.asarray(X, float).reshape(-1, self.dim))
        m = X.shape[0]
        J = np.zeros((m, 3))
        cnt = np.zeros(m, np.int32)
        h = self.handle()
        L = _lib.lib()
        _lib.check(L.vc_cache_set_blend(h, 1 if log_space else 0))
        _lib.check(L.vc_cache_interpolate(h, m, _lib.ptr(X), _lib.ptr(J), _lib.ptr(cnt), _lib.VC_MEM_HOST, None))
        return J, cnt


# Device mirrors of reference RadianceCache objects, dropped with them.  The reference
# cache is append-only (src/cache.py:298-315): a mirror whose last mirrored record is
# still in place only takes the new records; anything else is re-mirrored.
_MIRRORS: "weakref.WeakKeyDictionary" = weakref.WeakKeyDictionary()


def _ref_records(cache) -> list:
    recs = getattr(cache, "_records", None)
    return recs if isinstance(recs, list) else list(cache.records)


def _as_device_cache(cache) -> RadianceCache:
    """Accept a reference RadianceCache too: mirror its records on the device."""
    if isinstance(cache, RadianceCache):
        return cache
    recs = _ref_records(cache)
    n = len(recs)
    try:
        hit = _MIRRORS.get(cache)
    except TypeError:  # not weak-referenceable: no mirror kept
        return cache_from_records(cache.bounds_min, cache.bounds_max, recs)
    if hit is not None:
        m, last, dc = hit
        if n >= m and (m == 0 or recs[m - 1] is last):
            if n > m:
                dc._host_records().extend(cache_from_records(cache.bounds_min, cache.bounds_max, recs[m:])._records)
                _MIRRORS[cache] = (n, recs[-1], dc)
            return dc
    dc = cache_from_records(cache.bounds_min, cache.bounds_max, recs)
    _MIRRORS[cache] = (n, recs[-1] if n else None, dc)
    return dc


def interpolate(cache, x):
    """Cubic-weighted first-order blend of covering records, or None (src/cache.py:342-360)."""
    cache = _as_device_cache(cache)
    J, cnt = cache.interpolate_many(np.asarray(x, float)[None])
    if cnt[0] == 0 or np.isnan(J[0, 0]):
        return None
    return J[0]


def cache_from_records(bounds_min, bounds_max, records) -> RadianceCache:
    from .records import BaselineRecord

    c = RadianceCache(bounds_min, bounds_max)
    for r in records:
        if isinstance(r, (CacheRecord, BaselineRecord)):
            c._records.append(r)
        elif hasattr(r, "radius") and not hasattr(r, "axes"):  # reference BaselineRecord
            c._records.append(BaselineRecord(np.asarray(r.position, float), np.asarray(r.value, float),
                                             np.asarray(r.grad, float), float(r.radius)))
        else:
            c._records.append(CacheRecord(np.asarray(r.position, float), np.asarray(r.value, float),
                                          np.asarray(r.grad, float), np.asarray(r.axes, float),
                                          np.asarray(r.radii, float)))
    return c


def render_frozen(scene, camera: dict, single: RadianceCache, multiple: RadianceCache, *, spp=1,
                  march_step=0.1, seed=0, n_angular=None, n_inner=1, n_light_samples=16, epsilon=0.05,
                  crop=None):
    """Frozen-cache camera image (src/renderer.py:440-484) → (image (h, w, 3), stats).

    `camera` = {position, look_at, up, fov, width, height}; `crop` = (row0, rows, col0, cols)
    restricts the march to a pixel window (other pixels stay 0).  Misses are evaluated
    directly through the record build with seeds (seed, 211, k, i, m), as the reference.
    """
    ds = device_scene(scene)
    cam = _lib.Camera()
    for f in ("position", "look_at", "up"):
        getattr(cam, f)[:] = [float(v) for v in np.asarray(camera[f], float)]
    cam.fov_degrees = float(camera["fov"])
    cam.width = int(camera["width"])
    cam.height = int(camera["height"])
    if crop is not None:
        cam.row0, cam.rows, cam.col0, cam.cols = (int(v) for v in crop)
    rp = _lib.RenderParams()
    rp.spp = int(spp)
    rp.march_step = float(march_step)
    rp.seed = int(seed)
    rp.n_angular = int(16384 if n_angular is None else n_angular)
    rp.n_inner = int(n_inner)
    rp.n_light_samples = int(n_light_samples)
    rp.epsilon = float(epsilon)
    img = np.zeros((cam.height, cam.width, 3))
    stats = np.zeros(2, np.int64)
    _lib.check(_lib.lib().vc_render(ds.handle, single.handle(), multiple.handle(), _lib.C.byref(cam),
                                    _lib.C.byref(rp), _lib.ptr(img), _lib.ptr(stats), _lib.VC_MEM_HOST, None))
    return img, {"cache_hits": int(stats[0]), "direct_evaluations": int(stats[1])}
