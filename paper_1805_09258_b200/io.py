"""Cache files and images of the path, written from packed record rows.

Formats (the reference's, so files move freely between the two implementations):
* cache JSON — src/cache.py:397-491: {"format": "volcache-cache", "version": 1,
  "dimensionality", "bounds", "metadata", "records"} with "ellipsoid" (axes, radii) and
  "sphere" (radius) records, json indent 1 plus a trailing newline;
* binary sidecar — the device row layout (position, value, grad, axes,
  radii) plus creation tags, in one .npz;
* PFM (little-endian colour, bottom-up rows) and a tonemapped PPM — src/renderer.py:689-730.

Everything goes through the (N, d + 3 + 3d + d² + d) row matrix the device cache holds:
saving reads the rows once (vc_cache_records for a device-built cache) and emits the
document from them; loading validates the document into a row matrix and a kind vector
and builds the device cache in one call.
"""

from __future__ import annotations

import json

import numpy as np

from .cache import RadianceCache, _pack
from .records import BaselineRecord, CacheRecord, record_size

CACHE_FORMAT = "volcache-cache"
CACHE_VERSION = 1
_ELLIPSOID, _SPHERE = 0, 1


class CacheFormatError(ValueError):
    """A file that is not a version-1 volcache cache (src/cache.py:45-46)."""


def _layout(d: int) -> dict[str, slice]:
    """Field slices of a packed row."""
    o, out = 0, {}
    for name, k in (("position", d), ("value", 3), ("grad", 3 * d), ("axes", d * d), ("radii", d)):
        out[name] = slice(o, o + k)
        o += k
    return out


def _rows_and_kinds(cache) -> tuple[np.ndarray, np.ndarray]:
    """Packed rows + record kinds of a cache (host records, else the device rows)."""
    recs = cache._records if isinstance(cache, RadianceCache) else list(cache.records)
    if recs is None:  # held on the device only: the cache's mode decides the record type
        rows = cache.packed()
        kind = _SPHERE if getattr(cache, "sphere_records", False) else _ELLIPSOID
        return rows, np.full(len(rows), kind, np.int8)
    kinds = np.array([_SPHERE if (isinstance(r, BaselineRecord) or (hasattr(r, "radius") and not hasattr(r, "axes")))
                      else _ELLIPSOID for r in recs], np.int8)
    if len(kinds) and not np.all([hasattr(r, "position") for r in recs]):
        raise TypeError("unknown record type in cache")
    return _pack(recs, cache.dim), kinds


def _record_doc(row: np.ndarray, kind: int, f: dict, d: int) -> dict:
    doc = {"record_type": "sphere" if kind == _SPHERE else "ellipsoid",
           "position": row[f["position"]].tolist(), "value": row[f["value"]].tolist(),
           "grad": row[f["grad"]].reshape(3, d).tolist()}
    if kind == _SPHERE:
        doc["radius"] = float(row[f["radii"]][0])
    else:
        doc["axes"] = row[f["axes"]].reshape(d, d).tolist()
        doc["radii"] = row[f["radii"]].tolist()
    return doc


def save_cache(cache, path, metadata: dict | None = None) -> None:
    """Versioned JSON document of the cache's records, bounds and metadata."""
    d = cache.dim
    rows, kinds = _rows_and_kinds(cache)
    f = _layout(d)
    body = {
        "format": CACHE_FORMAT,
        "version": CACHE_VERSION,
        "dimensionality": d,
        "bounds": {"min": np.asarray(cache.bounds_min, float).tolist(),
                   "max": np.asarray(cache.bounds_max, float).tolist()},
        "metadata": metadata or {},
        "records": [_record_doc(r, int(k), f, d) for r, k in zip(rows, kinds)],
    }
    with open(path, "w", encoding="utf-8") as fh:
        fh.write(json.dumps(body, indent=1))
        fh.write("\n")


def _as_array(v, shape, what):
    try:
        a = np.asarray(v, dtype=float)
    except (TypeError, ValueError) as exc:
        raise CacheFormatError(f"malformed cache record: {what}: {exc}") from exc
    if a.shape != shape:
        raise CacheFormatError(f"cache record has inconsistent shapes ({what} {a.shape}, want {shape})")
    return a


def _parse_records(items, d: int) -> tuple[np.ndarray, np.ndarray]:
    if not isinstance(items, list):
        raise CacheFormatError("malformed cache file: records must be a list")
    f = _layout(d)
    rows = np.zeros((len(items), record_size(d)))
    kinds = np.zeros(len(items), np.int8)
    for i, it in enumerate(items):
        if not isinstance(it, dict):
            raise CacheFormatError("malformed cache record: not an object")
        for key in ("record_type", "position", "value", "grad"):
            if key not in it:
                raise CacheFormatError(f"malformed cache record: missing {key!r}")
        row = rows[i]
        row[f["position"]] = _as_array(it["position"], (d,), "position")
        row[f["value"]] = _as_array(it["value"], (3,), "value")
        row[f["grad"]] = _as_array(it["grad"], (3, d), "grad").ravel()
        rtype = it["record_type"]
        if rtype == "ellipsoid":
            if "axes" not in it or "radii" not in it:
                raise CacheFormatError("malformed cache record: ellipsoid without axes/radii")
            row[f["axes"]] = _as_array(it["axes"], (d, d), "axes").ravel()
            row[f["radii"]] = _as_array(it["radii"], (d,), "radii")
        elif rtype == "sphere":
            try:
                radius = float(it["radius"])
            except (KeyError, TypeError, ValueError) as exc:
                raise CacheFormatError(f"malformed cache record: radius: {exc}") from exc
            row[f["axes"]] = np.eye(d).ravel()
            row[f["radii"]] = radius
            kinds[i] = _SPHERE
        else:
            raise CacheFormatError(f"unknown record_type {rtype!r}")
    return rows, kinds


def _cache_from_rows(bmin, bmax, rows: np.ndarray, kinds: np.ndarray) -> RadianceCache:
    d = np.asarray(bmin).size
    f = _layout(d)
    cache = RadianceCache(bmin, bmax)
    recs = cache._records
    for row, k in zip(rows, kinds):
        p, v, g = row[f["position"]].copy(), row[f["value"]].copy(), row[f["grad"]].reshape(3, d).copy()
        if k == _SPHERE:
            recs.append(BaselineRecord(p, v, g, float(row[f["radii"]][0])))
        else:
            recs.append(CacheRecord(p, v, g, row[f["axes"]].reshape(d, d).copy(), row[f["radii"]].copy()))
    return cache


def load_cache(path) -> tuple[RadianceCache, dict]:
    """(cache, metadata) from a document written by save_cache (either implementation)."""
    try:
        with open(path, encoding="utf-8") as fh:
            doc = json.load(fh)
    except json.JSONDecodeError as exc:
        raise CacheFormatError(f"not a cache file: {exc}") from exc
    if not isinstance(doc, dict) or doc.get("format") != CACHE_FORMAT:
        raise CacheFormatError("not a radiance cache file")
    if doc.get("version") != CACHE_VERSION:
        raise CacheFormatError(f"unsupported cache version {doc.get('version')!r} (supported: {CACHE_VERSION})")
    try:
        d = int(doc["dimensionality"])
        bmin = np.asarray(doc["bounds"]["min"], dtype=float)
        bmax = np.asarray(doc["bounds"]["max"], dtype=float)
        items = doc["records"]
    except (KeyError, TypeError, ValueError) as exc:
        raise CacheFormatError(f"malformed cache file: {exc}") from exc
    if bmin.shape != (d,) or bmax.shape != (d,):
        if bmin.shape == bmax.shape and bmin.size in (2, 3):
            raise CacheFormatError("dimensionality does not match bounds")
        raise ValueError("bounds must be matching 2- or 3-vectors")
    rows, kinds = _parse_records(items, d)
    return _cache_from_rows(bmin, bmax, rows, kinds), doc.get("metadata", {})


def save_cache_npz(cache: RadianceCache, path, tags=None) -> None:
    """Binary sidecar: bounds, packed rows in the device layout, creation tags."""
    rows, kinds = _rows_and_kinds(cache)
    np.savez(path, format=np.array(CACHE_FORMAT), version=np.array(CACHE_VERSION),
             bounds_min=np.asarray(cache.bounds_min, float), bounds_max=np.asarray(cache.bounds_max, float),
             records=rows, kinds=kinds,
             tags=np.asarray(tags if tags is not None else np.full(len(rows), -1), np.int64))


def load_cache_npz(path) -> RadianceCache:
    z = np.load(path, allow_pickle=False)
    if str(z["format"]) != CACHE_FORMAT or int(z["version"]) != CACHE_VERSION:
        raise CacheFormatError("not a radiance cache sidecar")
    bmin, bmax = z["bounds_min"], z["bounds_max"]
    rows = np.asarray(z["records"], float).reshape(-1, record_size(bmin.size)) if z["records"].size else \
        np.zeros((0, record_size(bmin.size)))
    if z["records"].size and z["records"].shape[1] != record_size(bmin.size):
        raise CacheFormatError("sidecar rows do not match the dimensionality")
    kinds = z["kinds"] if "kinds" in z.files else np.zeros(len(rows), np.int8)
    return _cache_from_rows(bmin, bmax, rows, kinds)


# ---------------------------------------------------------------------------
# Images
# ---------------------------------------------------------------------------


def _rgb_image(image, dtype, who):
    a = np.asarray(image, dtype=dtype)
    if a.ndim != 3 or a.shape[2] != 3:
        raise ValueError(f"{who} expects an (h, w, 3) image")
    return a


def write_pfm(path, image: np.ndarray) -> None:
    """Colour PFM, little endian (scale −1), rows stored bottom-up; row 0 of `image` is the top."""
    a = _rgb_image(image, np.float32, "write_pfm")
    h, w = a.shape[:2]
    header = b"PF\n%d %d\n-1.0\n" % (w, h)
    with open(path, "wb") as fh:
        fh.write(header + np.ascontiguousarray(np.flipud(a), dtype="<f4").tobytes())


def read_pfm(path):
    """(h, w, 3) float32 image, row 0 = top, from a colour PFM of either endianness."""
    with open(path, "rb") as fh:
        raw = fh.read()
    parts = raw.split(b"\n", 3)
    if len(parts) < 4 or parts[0].strip() != b"PF":
        raise ValueError("not a color PFM file")
    w, h = (int(v) for v in parts[1].split())
    endian = "<" if float(parts[2]) < 0 else ">"
    data = np.frombuffer(parts[3], dtype=endian + "f4")
    if data.size != w * h * 3:
        raise ValueError("PFM payload size mismatch")
    return np.flipud(data.reshape(h, w, 3)).astype(np.float32)


def write_ppm(path, image: np.ndarray, exposure: float = 1.0) -> None:
    """8-bit binary PPM after exposure, clipping to [0, 1] and gamma 1/2.2 (for quick looks)."""
    a = _rgb_image(image, float, "write_ppm")
    q = (np.clip(a * exposure, 0.0, 1.0) ** (1.0 / 2.2) * 255.0 + 0.5).astype(np.uint8)
    h, w = a.shape[:2]
    with open(path, "wb") as fh:
        fh.write(b"P6\n%d %d\n255\n" % (w, h) + q.tobytes())
