"""Occlusion-unaware baseline estimator and its log-space cache on the B200 path.

Drop-ins for baseline_estimate / occlusion_unaware_gradient (src/subdivision.py:401-536),
log_gradient_radius / make_baseline_record (src/cache.py:190-226) and
log_space_interpolate (src/cache.py:363-394).  The per-direction paths, the rigid-path
derivatives and the reductions run in libvolcache_b200.so (vc_baseline_records); the
log-space blend runs in the cache lookup kernel (vc_cache_set_blend).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .records import BaselineRecord
from .records import DEFAULT_N_ANGULAR, device_scene, pcg64_state, record_size

R_MAX_FRACTION = 0.25  # src/cache.py:30
R_MIN_FRACTION = 1e-3  # src/cache.py:33


@dataclass(frozen=True)
class BaselineEstimate:
    """Value + gradient of the fixed-hit-point estimator (src/subdivision.py:401-414)."""

    value: np.ndarray
    grad: np.ndarray
    sample_values: np.ndarray
    sample_grad_norms: np.ndarray
    kind: str


def _bparams(n_angular, max_media_bounces, n_light_samples, alpha, flags, seed_words=0):
    p = _lib.BaselineParams()
    p.n_angular = int(n_angular)
    p.max_media_bounces = int(max_media_bounces)
    p.n_light_samples = int(n_light_samples)
    p.alpha = float(alpha)
    p.flags = int(flags)
    p.seed_words = int(seed_words)
    return p


def baseline_estimate(scene, x, n_angular=None, rng_seed=None, max_media_bounces=2, n_light_samples=16):
    """(single, multiple) BaselineEstimate at x (src/subdivision.py:416-509)."""
    ds = device_scene(scene)
    d = ds.dim
    x = np.ascontiguousarray(np.asarray(x, float).reshape(-1))
    if x.size != d:
        raise ValueError("x dimensionality does not match the scene")
    n = int(DEFAULT_N_ANGULAR[d] if n_angular is None else n_angular)
    st, gen = pcg64_state(rng_seed)
    p = _bparams(n, max_media_bounces, n_light_samples, 1.0, _lib.VC_MEM_HOST)
    draws = np.zeros(1, np.int64)
    p.draws = draws.ctypes.data
    es = 3 + 3 * d
    est = np.zeros((2, es))
    smp = np.zeros((2, 2, n))
    _lib.check(_lib.lib().vc_baseline_records(ds.handle, 1, _lib.ptr(x), _lib.ptr(st), _lib.C.byref(p),
                                              _lib.ptr(est), None, _lib.ptr(smp), None))
    if isinstance(rng_seed, np.random.Generator):  # default_rng(gen) hands back gen itself
        gen.bit_generator.advance(int(draws[0]))
    out = []
    for k, kind in enumerate(("single", "multiple")):
        out.append(BaselineEstimate(value=est[k, :3].copy(), grad=est[k, 3:].reshape(3, d).copy(),
                                    sample_values=smp[k, 0].copy(), sample_grad_norms=smp[k, 1].copy(), kind=kind))
    return out[0], out[1]


def occlusion_unaware_gradient(scene, x, n_angular=None, rng_seed=None, max_media_bounces=2, n_light_samples=16):
    """(single, multiple) gradients of the baseline (src/subdivision.py:524-536)."""
    s, m = baseline_estimate(scene, x, n_angular=n_angular, rng_seed=rng_seed, max_media_bounces=max_media_bounces,
                             n_light_samples=n_light_samples)
    return s.grad, m.grad


def log_gradient_radius(sample_values, sample_grad_norms, scene_scale: float, alpha: float = 1.0) -> float:
    """α·ΣLⱼ/Σ‖∇Lⱼ‖ clamped to [R_MIN, R_MAX]·scale (src/cache.py:190-209)."""
    num = float(np.sum(sample_values))
    den = float(np.sum(sample_grad_norms))
    r_max = R_MAX_FRACTION * scene_scale
    if den <= 0.0:
        return r_max
    return float(np.clip(alpha * num / den, R_MIN_FRACTION * scene_scale, r_max))


def make_baseline_record(x, estimate: BaselineEstimate, scene_scale: float, alpha: float = 1.0) -> BaselineRecord:
    """src/cache.py:212-226."""
    x = np.asarray(x, dtype=float)
    radius = log_gradient_radius(estimate.sample_values, estimate.sample_grad_norms, scene_scale, alpha)
    return BaselineRecord(position=x, value=np.asarray(estimate.value, float).copy(),
                          grad=np.asarray(estimate.grad, float).copy(), radius=radius)


def baseline_records_batch(scene, X, seeds, n_angular=None, max_media_bounces=2, n_light_samples=16, alpha=1.0):
    """N baseline record pairs in one call → (estimates (N, 2, 3+3d), records (N, 2, row))."""
    ds = device_scene(scene)
    d = ds.dim
    X = np.ascontiguousarray(np.asarray(X, float).reshape(-1, d))
    N = X.shape[0]
    words = np.ascontiguousarray(np.asarray(seeds, np.uint32).reshape(N, -1))
    n = int(DEFAULT_N_ANGULAR[d] if n_angular is None else n_angular)
    p = _bparams(n, max_media_bounces, n_light_samples, alpha, _lib.VC_MEM_HOST | _lib.VC_SEED_WORDS,
                 words.shape[1])
    est = np.zeros((N, 2, 3 + 3 * d))
    rec = np.zeros((N, 2, record_size(d)))
    if N:
        _lib.check(_lib.lib().vc_baseline_records(ds.handle, N, _lib.ptr(X), _lib.ptr(words), _lib.C.byref(p),
                                                  _lib.ptr(est), _lib.ptr(rec), None, None))
    return est, rec


def log_space_interpolate(cache, x):
    """Log-space blend exp(Σw(ln L + ∇L·Δ/L)/Σw), or None (src/cache.py:363-394)."""
    from .cache import _as_device_cache

    cache = _as_device_cache(cache)
    J, cnt = cache.interpolate_many(np.asarray(x, float)[None], log_space=True)
    if cnt[0] == 0 or np.isnan(J[0, 0]):
        return None
    return J[0]
