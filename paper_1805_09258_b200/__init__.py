"""volcache on B200: the cache-record build and lookup path of arXiv 1805.09258.

Public API mirrors the reference `volcache` entry points for this path
(estimate_moments, make_record, RadianceCache, interpolate, frozen camera render),
backed by hand-written sm_100a kernels in libvolcache_b200.so (C ABI:
include/volcache_b200.h).  There is no CPU fallback.
"""

from .cache import RadianceCache, cache_from_records, interpolate, render_frozen
from .records import (
    DEFAULT_N_ANGULAR,
    BatchResult,
    CacheRecord,
    DeviceScene,
    Moments,
    device_scene,
    estimate_moments,
    estimate_moments_batch,
    inspect_record,
    make_record,
    make_records,
    seed_words,
)
from .scene import Medium, Scene, Surface, load_scene, save_scene

__all__ = [
    "DEFAULT_N_ANGULAR", "BatchResult", "CacheRecord", "DeviceScene", "Moments", "RadianceCache",
    "Medium", "Scene", "Surface", "cache_from_records", "device_scene", "estimate_moments",
    "estimate_moments_batch", "inspect_record", "interpolate", "load_scene", "make_record",
    "make_records", "render_frozen", "save_scene", "seed_words",
]
