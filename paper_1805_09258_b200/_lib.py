"""ctypes binding of libvolcache_b200.so (the C ABI in include/volcache_b200.h).

There is no fallback: if the shared library is missing or no CUDA device is usable,
every entry point raises.  Error codes map to the reference's exception types:
VC_EINVAL / VC_EOUTSIDE → ValueError (src/subdivision.py:155-158), others → RuntimeError.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(os.environ.get("VOLCACHE_B200_LIB", Path(__file__).resolve().parent / "lib" / "libvolcache_b200.so"))

VC_OK = 0
VC_EINVAL = -1
VC_EOUTSIDE = -2
VC_ECUDA = -3
VC_ETRI = -4
VC_ENOMEM = -5
VC_EHOOK = -6

VC_MEM_HOST = 1
VC_SEED_WORDS = 2
VC_MAKE_RECORDS = 4
VC_ISOTROPIC = 8
VC_DEFER_CHECK = 32
VC_TRACE_BOUNDS = 16

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_lp = C.POINTER(C.c_int64)
_vp = C.c_void_p


class BuildParams(C.Structure):
    _fields_ = [
        ("n_angular", C.c_int),
        ("march_step", C.c_double),
        ("n_inner", C.c_int),
        ("n_light_samples", C.c_int),
        ("epsilon", C.c_double),
        ("flags", C.c_int),
        ("seed_words", C.c_int),
        ("media_bounces", C.c_int),
        ("hg_g", C.c_double),
    ]


class Camera(C.Structure):
    _fields_ = [
        ("position", C.c_double * 3),
        ("look_at", C.c_double * 3),
        ("up", C.c_double * 3),
        ("fov_degrees", C.c_double),
        ("width", C.c_int),
        ("height", C.c_int),
        ("row0", C.c_int),
        ("rows", C.c_int),
        ("col0", C.c_int),
        ("cols", C.c_int),
    ]


class RenderParams(C.Structure):
    _fields_ = [
        ("spp", C.c_int),
        ("march_step", C.c_double),
        ("seed", C.c_int),
        ("n_angular", C.c_int),
        ("n_inner", C.c_int),
        ("n_light_samples", C.c_int),
        ("epsilon", C.c_double),
        ("estimator", C.c_int),
        ("max_media_bounces", C.c_int),
        ("path_samples", C.c_int),
        ("grow", C.c_int),
        ("isotropic", C.c_int),
        ("baseline_alpha", C.c_double),
    ]


VC_EST_SUBDIVISION = 0
VC_EST_BASELINE = 1
VC_EST_PATH = 2
VC_TARGET_FIELD = 1
VC_TARGET_CAMERA = 2


class PopulateParams(C.Structure):
    _fields_ = [
        ("target", C.c_int),
        ("camera", Camera),
        ("field_nx", C.c_int),
        ("field_ny", C.c_int),
        ("field_min", C.c_double * 2),
        ("field_max", C.c_double * 2),
        ("march_step", C.c_double),
        ("seed", C.c_int),
        ("n_angular", C.c_int),
        ("n_inner", C.c_int),
        ("n_light_samples", C.c_int),
        ("epsilon", C.c_double),
        ("isotropic", C.c_int),
        ("window", C.c_int),
        ("lookahead", C.c_int64),
        ("estimator", C.c_int),
        ("max_media_bounces", C.c_int),
        ("baseline_alpha", C.c_double),
        ("path_samples", C.c_int),
        ("build_hook", C.c_void_p),
        ("build_hook_user", C.c_void_p),
    ]


# int (*)(void* user, int n, const double* x, const uint32_t* words, int seed_words,
#         double* rec_out, int64_t* stats_out, void* stream)
BUILD_HOOK = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p,
                         C.c_void_p)


class BaselineParams(C.Structure):
    _fields_ = [
        ("n_angular", C.c_int),
        ("max_media_bounces", C.c_int),
        ("n_light_samples", C.c_int),
        ("alpha", C.c_double),
        ("flags", C.c_int),
        ("seed_words", C.c_int),
        ("draws", C.c_void_p),
    ]


_SIGS = {
    "vc_version": (C.c_int, []),
    "vc_last_error": (C.c_char_p, []),
    "vc_kernel_launches": (C.c_int64, []),
    "vc_profile": (C.c_int, [C.c_int]),
    "vc_profile_read": (C.c_int, [_vp, _vp, C.c_int]),
    "vc_scene_create": (C.c_int, [C.c_int, C.c_int, _vp, _vp, _vp, _vp, _vp, C.c_double, C.c_double,
                                  C.POINTER(_vp)]),
    "vc_scene_destroy": (None, [_vp]),
    "vc_scene_set_budget": (C.c_int, [_vp, C.c_int64]),
    "vc_check_deferred": (C.c_int, [_vp]),
    "vc_scene_set_lights": (C.c_int, [_vp, C.c_int, _vp]),
    "vc_build_records": (C.c_int, [_vp, C.c_int, _vp, _vp, _vp, C.POINTER(BuildParams), _vp, _vp, _vp, _vp]),
    "vc_build_inspect": (C.c_int, [_vp, _vp, _vp, _vp, C.POINTER(BuildParams), _vp, _vp, _vp, _vp, _vp, _vp,
                                   C.c_int64, _vp, _vp, _vp]),
    "vc_make_records": (C.c_int, [C.c_int, C.c_int, _vp, _vp, C.c_double, C.c_double, C.c_double, C.c_int,
                                  _vp, _vp]),
    "vc_trace": (C.c_int, [_vp, C.c_int, _vp, _vp, _vp, _vp, C.c_int, _vp]),
    "vc_surface_radiance": (C.c_int, [_vp, C.c_int, _vp, _vp, _vp, C.c_int, _vp, C.c_int, _vp]),
    "vc_seed_states": (C.c_int, [C.c_int, _vp, C.c_int, _vp]),
    "vc_cache_create": (C.c_int, [C.c_int, _vp, _vp, C.c_int, _vp, C.POINTER(_vp)]),
    "vc_cache_destroy": (None, [_vp]),
    "vc_cache_insert": (C.c_int, [_vp, C.c_int, _vp, C.c_int, _vp]),
    "vc_form_factors": (C.c_int, [C.c_int, C.c_int, _vp, _vp, C.c_int, C.c_int, _vp, _vp, _vp, _vp, _vp]),
    "vc_cache_interpolate": (C.c_int, [_vp, C.c_int, _vp, _vp, _vp, C.c_int, _vp]),
    "vc_render": (C.c_int, [_vp, _vp, _vp, C.POINTER(Camera), C.POINTER(RenderParams), _vp, _vp, C.c_int, _vp]),
    "vc_cache_size": (C.c_int64, [_vp]),
    "vc_cache_set_blend": (C.c_int, [_vp, C.c_int]),
    "vc_path_trace": (C.c_int, [_vp, C.c_int, _vp, _vp, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int, _vp, _vp]),
    "vc_baseline_records": (C.c_int, [_vp, C.c_int, _vp, _vp, C.POINTER(BaselineParams), _vp, _vp, _vp, _vp]),
    "vc_cache_records": (C.c_int, [_vp, _vp, _vp, C.c_int, _vp]),
    "vc_populate": (C.c_int, [_vp, C.POINTER(PopulateParams), C.POINTER(_vp), C.POINTER(_vp), _vp, _vp]),
    "vc_render_field": (C.c_int, [_vp, _vp, _vp, C.POINTER(PopulateParams), C.c_int, _vp, _vp, C.c_int, _vp]),
}

EXPORTS = tuple(_SIGS)

KERNEL_CLASSES = ("primary", "rings", "wave_scan", "gather", "delaunay", "tri_compact", "degree",
                  "assemble", "make_record", "seedseq", "interpolate", "march")

_lib = None


def lib():
    """Load (once) and return the shared library; raises if it is not built."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)"
            )
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc == VC_OK:
        return
    msg = lib().vc_last_error().decode(errors="replace")
    if rc in (VC_EINVAL, VC_EOUTSIDE):
        raise ValueError(msg)
    raise RuntimeError(f"libvolcache_b200 error {rc}: {msg}")


def ptr(a):
    """Address of a numpy array or torch tensor (None → NULL)."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.ctypes.data
