"""Path-traced reference estimator and finite-difference derivative oracle on the B200 path.

Drop-ins for path_trace_radiance (src/transport.py:318-391) and fd_derivatives /
TransportDerivativeEstimate (src/renderer.py:584-649).  All samples of all evaluation
points run in one vc_path_trace call; every point of an FD stencil reuses the same
PCG64 stream, which is exactly the reference's common-random-number construction.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .records import device_scene, pcg64_state


@dataclass(frozen=True)
class TransportDerivativeEstimate:
    """src/renderer.py:584-587."""

    value: np.ndarray
    grad: np.ndarray
    hess: np.ndarray | None


def _trace_points(scene, X, n_samples, max_media_bounces, rng_seed, n_light_samples):
    ds = device_scene(scene)
    X = np.ascontiguousarray(np.asarray(X, float).reshape(-1, ds.dim))
    st, _ = pcg64_state(rng_seed)
    rng = np.ascontiguousarray(np.broadcast_to(st, (X.shape[0], 4)))
    out = np.zeros((X.shape[0], 2, 3))
    _lib.check(_lib.lib().vc_path_trace(ds.handle, X.shape[0], _lib.ptr(X), _lib.ptr(rng), int(n_samples),
                                        int(max_media_bounces), int(n_light_samples), _lib.VC_MEM_HOST, 0,
                                        _lib.ptr(out), None))
    return out


def path_trace_radiance(scene, x, n_samples, max_media_bounces=2, rng_seed=None, n_light_samples=16):
    """Unbiased MC (J_single, J_multiple) at a media point (src/transport.py:318-391)."""
    out = _trace_points(scene, np.asarray(x, float)[None], n_samples, max_media_bounces, rng_seed, n_light_samples)
    return out[0, 0].copy(), out[0, 1].copy()


def _unit(dim: int, i: int) -> np.ndarray:
    e = np.zeros(dim)
    e[i] = 1.0
    return e


def fd_derivatives(scene, x, h, n_samples, seed=0, max_media_bounces=2, include_hessian=False,
                   n_light_samples=16):
    """Central finite differences of path-traced J with common random numbers
    (src/renderer.py:590-643) → (single, multiple) TransportDerivativeEstimate."""
    x = np.asarray(x, dtype=float)
    dim = x.size
    pts = [x]
    pts += [x + h * _unit(dim, i) for i in range(dim)]
    pts += [x - h * _unit(dim, i) for i in range(dim)]
    pairs = []
    if include_hessian:
        for i in range(dim):
            for j in range(i + 1, dim):
                ei, ej = h * _unit(dim, i), h * _unit(dim, j)
                pairs.append((i, j, len(pts)))
                pts += [x + ei + ej, x + ei - ej, x - ei + ej, x - ei - ej]
    vals = _trace_points(scene, np.array(pts), n_samples, max_media_bounces, seed, n_light_samples)
    base = vals[0]
    plus = vals[1:1 + dim]
    minus = vals[1 + dim:1 + 2 * dim]
    out = []
    for part in range(2):
        value = base[part].copy()
        grad = np.stack([(plus[i][part] - minus[i][part]) / (2.0 * h) for i in range(dim)], axis=1)
        hess = None
        if include_hessian:
            hess = np.zeros((3, dim, dim))
            for i in range(dim):
                hess[:, i, i] = (plus[i][part] - 2.0 * value + minus[i][part]) / h**2
            for i, j, k in pairs:
                pp, pm, mp, mm = (vals[k + q][part] for q in range(4))
                hess[:, i, j] = hess[:, j, i] = (pp - pm - mp + mm) / (4.0 * h**2)
        out.append(TransportDerivativeEstimate(value=value, grad=grad, hess=hess))
    return out[0], out[1]
