"""On-disk formats of the path: cache JSON (+ a binary SoA sidecar) and PFM/PPM images.

save_cache / load_cache write and read the reference's versioned JSON document
(src/cache.py:397-491: format "volcache-cache", version 1, ellipsoid and sphere
records), so caches built on the GPU load in the reference's tools and vice versa.
save_cache_npz / load_cache_npz are the binary sidecar: packed
record rows in the device layout plus the creation tags of a populated cache.
write_pfm / read_pfm / write_ppm follow src/renderer.py:689-730.
"""

from __future__ import annotations

import json
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from .cache import RadianceCache
from .records import CacheRecord, record_size, unpack_record

CACHE_FORMAT = "volcache-cache"
CACHE_VERSION = 1


class CacheFormatError(ValueError):
    """Raised for malformed or version-incompatible cache files (src/cache.py:45-46)."""


@dataclass(frozen=True)
class BaselineRecord:
    """Value + gradient with an isotropic valid region (src/cache.py:124-145).

    Stored and indexed on the device as an ellipsoid with identity axes and equal radii.
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


def _record_to_dict(rec) -> dict:
    if isinstance(rec, BaselineRecord):
        return {"record_type": "sphere", "position": np.asarray(rec.position, float).tolist(),
                "value": np.asarray(rec.value, float).tolist(), "grad": np.asarray(rec.grad, float).tolist(),
                "radius": float(rec.radius)}
    if isinstance(rec, CacheRecord) or hasattr(rec, "axes"):
        return {"record_type": "ellipsoid", "position": np.asarray(rec.position, float).tolist(),
                "value": np.asarray(rec.value, float).tolist(), "grad": np.asarray(rec.grad, float).tolist(),
                "axes": np.asarray(rec.axes, float).tolist(), "radii": np.asarray(rec.radii, float).tolist()}
    raise TypeError(f"unknown record type {type(rec)!r}")


def _record_from_dict(d: dict, dim: int):
    try:
        rtype = d["record_type"]
        position = np.asarray(d["position"], dtype=float)
        value = np.asarray(d["value"], dtype=float)
        grad = np.asarray(d["grad"], dtype=float)
    except (KeyError, TypeError, ValueError) as exc:
        raise CacheFormatError(f"malformed cache record: {exc}") from exc
    if position.shape != (dim,) or value.shape != (3,) or grad.shape != (3, dim):
        raise CacheFormatError("cache record has inconsistent shapes")
    if rtype == "ellipsoid":
        try:
            axes = np.asarray(d["axes"], dtype=float)
            radii = np.asarray(d["radii"], dtype=float)
        except (KeyError, TypeError, ValueError) as exc:
            raise CacheFormatError(f"malformed cache record: {exc}") from exc
        if axes.shape != (dim, dim) or radii.shape != (dim,):
            raise CacheFormatError("cache record has inconsistent shapes")
        return CacheRecord(position=position, value=value, grad=grad, axes=axes, radii=radii)
    if rtype == "sphere":
        try:
            radius = float(d["radius"])
        except (KeyError, TypeError, ValueError) as exc:
            raise CacheFormatError(f"malformed cache record: {exc}") from exc
        return BaselineRecord(position=position, value=value, grad=grad, radius=radius)
    raise CacheFormatError(f"unknown record_type {rtype!r}")


def save_cache(cache: RadianceCache, path, metadata: dict | None = None) -> None:
    """Write the cache to versioned JSON (records, bounds, optional metadata)."""
    doc = {
        "format": CACHE_FORMAT,
        "version": CACHE_VERSION,
        "dimensionality": cache.dim,
        "bounds": {"min": cache.bounds_min.tolist(), "max": cache.bounds_max.tolist()},
        "metadata": metadata or {},
        "records": [_record_to_dict(r) for r in cache.records],
    }
    with open(path, "w", encoding="utf-8") as fh:
        json.dump(doc, fh, indent=1)
        fh.write("\n")


def load_cache(path) -> tuple[RadianceCache, dict]:
    """Read a cache written by save_cache (either implementation); returns (cache, metadata)."""
    with open(path, encoding="utf-8") as fh:
        try:
            doc = json.load(fh)
        except json.JSONDecodeError as exc:
            raise CacheFormatError(f"not a cache file: {exc}") from exc
    if not isinstance(doc, dict) or doc.get("format") != CACHE_FORMAT:
        raise CacheFormatError("not a radiance cache file")
    version = doc.get("version")
    if version != CACHE_VERSION:
        raise CacheFormatError(f"unsupported cache version {version!r} (supported: {CACHE_VERSION})")
    try:
        dim = int(doc["dimensionality"])
        bounds_min = np.asarray(doc["bounds"]["min"], dtype=float)
        bounds_max = np.asarray(doc["bounds"]["max"], dtype=float)
        record_dicts = doc["records"]
    except (KeyError, TypeError, ValueError) as exc:
        raise CacheFormatError(f"malformed cache file: {exc}") from exc
    cache = RadianceCache(bounds_min, bounds_max)
    if cache.dim != dim:
        raise CacheFormatError("dimensionality does not match bounds")
    for d in record_dicts:
        cache.insert(_record_from_dict(d, dim))
    return cache, doc.get("metadata", {})


def save_cache_npz(cache: RadianceCache, path, tags=None) -> None:
    """Binary SoA sidecar: bounds + packed rows (d + 3 + 3d + d² + d float64 each)."""
    np.savez(path, format=np.array(CACHE_FORMAT), version=np.array(CACHE_VERSION),
             bounds_min=cache.bounds_min, bounds_max=cache.bounds_max, records=cache.packed(),
             tags=np.asarray(tags if tags is not None else np.full(len(cache), -1), np.int64))


def load_cache_npz(path) -> RadianceCache:
    z = np.load(path, allow_pickle=False)
    if str(z["format"]) != CACHE_FORMAT or int(z["version"]) != CACHE_VERSION:
        raise CacheFormatError("not a radiance cache sidecar")
    cache = RadianceCache(z["bounds_min"], z["bounds_max"])
    rows = np.asarray(z["records"], float)
    if rows.size and rows.shape[1] != record_size(cache.dim):
        raise CacheFormatError("sidecar rows do not match the dimensionality")
    for r in rows:
        cache.insert(unpack_record(r, cache.dim))
    return cache


def write_pfm(path, image: np.ndarray) -> None:
    """Write a (h, w, 3) float image (row 0 = top) as a little-endian color PFM."""
    image = np.asarray(image, dtype=np.float32)
    if image.ndim != 3 or image.shape[2] != 3:
        raise ValueError("write_pfm expects an (h, w, 3) image")
    h, w = image.shape[:2]
    with open(path, "wb") as fh:
        fh.write(b"PF\n")
        fh.write(f"{w} {h}\n".encode("ascii"))
        fh.write(b"-1.0\n")
        fh.write(image[::-1].astype("<f4").tobytes())  # PFM rasters are bottom-up


def read_pfm(path):
    """Read a color PFM; returns (h, w, 3) float32 with row 0 = top."""
    with open(Path(path), "rb") as fh:
        if fh.readline().strip() != b"PF":
            raise ValueError("not a color PFM file")
        w, h = (int(v) for v in fh.readline().split())
        scale = float(fh.readline())
        data = np.frombuffer(fh.read(), dtype="<f4" if scale < 0 else ">f4")
    if data.size != w * h * 3:
        raise ValueError("PFM payload size mismatch")
    return data.reshape(h, w, 3)[::-1].astype(np.float32)


def write_ppm(path, image: np.ndarray, exposure: float = 1.0) -> None:
    """Gamma-2.2 tonemapped 8-bit PPM for quick looks."""
    image = np.asarray(image, dtype=float)
    if image.ndim != 3 or image.shape[2] != 3:
        raise ValueError("write_ppm expects an (h, w, 3) image")
    mapped = np.clip(image * exposure, 0.0, 1.0) ** (1.0 / 2.2)
    bytes8 = (mapped * 255.0 + 0.5).astype(np.uint8)
    h, w = image.shape[:2]
    with open(path, "wb") as fh:
        fh.write(f"P6\n{w} {h}\n255\n".encode("ascii"))
        fh.write(bytes8.tobytes())
