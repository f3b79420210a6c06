"""volcache on B200: the cache-record build and lookup path of arXiv 1805.09258.

Public API mirrors the reference `volcache` entry points for this path
(estimate_moments, make_record, RadianceCache, interpolate, populate_cache, render,
save_cache / load_cache, PFM I/O),
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
    check_deferred,
    device_scene,
    estimate_moments,
    estimate_moments_batch,
    inspect_record,
    make_record,
    make_records,
    seed_words,
    surface_radiance_batch,
)
from .io import (CACHE_FORMAT, CACHE_VERSION, BaselineRecord, CacheFormatError, load_cache, load_cache_npz, read_pfm,
                 save_cache, save_cache_npz, write_pfm, write_ppm)
from .renderer import (CACHE_MODES, MODES, CacheSet, Camera, FieldGrid, RenderSettings, populate_cache, render)
from .scene import Medium, Scene, Surface, directional_light, load_scene, point_light, save_scene
from . import baseline, path  # noqa: E402  (submodules: b200.baseline.*, b200.path.*)
from .baseline import (BaselineEstimate, baseline_estimate, log_gradient_radius, log_space_interpolate,
                       make_baseline_record, occlusion_unaware_gradient)
from .path import TransportDerivativeEstimate, fd_derivatives, path_trace_radiance

__all__ = [
    "CACHE_FORMAT", "CACHE_MODES", "CACHE_VERSION", "MODES", "BaselineRecord", "CacheFormatError", "CacheSet",
    "Camera", "FieldGrid", "RenderSettings", "load_cache", "load_cache_npz", "populate_cache", "read_pfm", "render",
    "save_cache", "save_cache_npz", "write_pfm", "write_ppm",
    "BaselineEstimate", "TransportDerivativeEstimate", "baseline_estimate", "fd_derivatives", "log_gradient_radius",
    "log_space_interpolate", "make_baseline_record", "occlusion_unaware_gradient", "path_trace_radiance",
    "DEFAULT_N_ANGULAR", "BatchResult", "CacheRecord", "DeviceScene", "Moments", "RadianceCache",
    "Medium", "Scene", "Surface", "cache_from_records", "check_deferred", "device_scene", "estimate_moments",
    "estimate_moments_batch", "inspect_record", "interpolate", "load_scene", "make_record",
    "make_records", "render_frozen", "save_scene", "seed_words", "surface_radiance_batch",
]
