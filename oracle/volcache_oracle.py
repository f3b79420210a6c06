"""CPU oracle for the cache-record hot path — TEST INFRASTRUCTURE ONLY.

This module is a numpy restatement of the reference `volcache` algorithm for the
path named in BASELINE.json:north_star (record build → make_record → lookup →
camera march).  It exists to check the CUDA product path; the product never
imports it.  Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs may call it.

Parity pin: `tests/golden/make_goldens.py` runs the real reference (imported
read-only from /root/reference/pkg/src in the build container) and stores its
outputs as fixtures; `tests/test_oracle_golden.py` checks this restatement
against them (bit-for-bit on integer data, ≤1e-12 relative on float data).

Reference citations use `src/` = /root/reference/pkg/src/volcache/.

Third-party dependencies restated or used here (not vendored by the reference):
* numpy PCG64 + SeedSequence (`numpy>=1.24`, pkg/pyproject.toml:10-13; container
  numpy 2.3.5) — used as is via `np.random.default_rng`, exactly as the reference.
* scipy.spatial.ConvexHull / qhull (`scipy>=1.10`; container scipy 1.18.1) for
  3D stratum connectivity (src/scene.py:388-399) — used as is; the
  `adjacency=` hook injects a different triangle list (the GPU's canonical
  spherical Delaunay) so arithmetic can be compared independently of qhull's
  vertex order.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# --- constants (src/scene.py:22-24, src/formfactor.py:23-30, src/cache.py:29-42) ---
T_EPS_REL = 1e-6
LUMA = np.array([0.2126, 0.7152, 0.0722])
GAMMA_MIN = 1e-5
A_REL_MIN = 1e-12
R_MAX_FRACTION = 0.25
L_FLOOR_FRACTION = 1e-6
CURVATURE_FLOOR = 1e-12
TREE_MAX_DEPTH = 16
CHUNK = 1 << 16  # src/transport.py:34


# ---------------------------------------------------------------------------
# Scene view (duck-typed over the reference Scene or the package mirror)
# ---------------------------------------------------------------------------


@dataclass
class PackedScene:
    """Flat float64 arrays of a scene, as `_Packed2D/_Packed3D` (src/scene.py:124-143)."""

    dim: int
    verts: np.ndarray  # (K, k, dim)
    emission: np.ndarray  # (K, 3)
    albedo: np.ndarray  # (K, 3)
    bmin: np.ndarray
    bmax: np.ndarray
    sigma_s: float
    sigma_a: float
    # extension (not in the reference): delta lights, rows (kind, v0, v1, v2, r, g, b, 0) —
    # kind 0 = point light at v with radiant intensity rgb, kind 1 = directional light whose
    # unit vector v points TOWARD the light, with irradiance rgb on a plane facing it
    lights: np.ndarray = field(default_factory=lambda: np.zeros((0, 8)))
    # derived (+ cached flat primitive array for the C helper)
    _prim: np.ndarray = field(init=False, default=None, repr=False)
    a: np.ndarray = field(init=False)
    e1: np.ndarray = field(init=False)
    e2: np.ndarray = field(init=False)
    normal: np.ndarray = field(init=False)

    def __post_init__(self):
        K = self.verts.shape[0]
        if self.dim == 2:
            self.a = self.verts[:, 0].reshape(K, 2)
            self.e1 = (self.verts[:, 1] - self.verts[:, 0]).reshape(K, 2)
            self.e2 = np.zeros((K, 2))
            ln = np.linalg.norm(self.e1, axis=1)
            self.normal = np.column_stack([-self.e1[:, 1], self.e1[:, 0]]) / ln[:, None]
        else:
            self.a = self.verts[:, 0].reshape(K, 3)
            self.e1 = (self.verts[:, 1] - self.verts[:, 0]).reshape(K, 3)
            self.e2 = (self.verts[:, 2] - self.verts[:, 0]).reshape(K, 3)
            nrm = np.cross(self.e1, self.e2)
            self.normal = nrm / np.linalg.norm(nrm, axis=1)[:, None]

    @property
    def K(self) -> int:
        return self.verts.shape[0]

    @property
    def sigma_t(self) -> float:
        return self.sigma_s + self.sigma_a

    @property
    def scale(self) -> float:  # src/scene.py:179-182
        return float(np.linalg.norm(self.bmax - self.bmin))

    @property
    def max_emission(self) -> float:  # src/scene.py:184-188
        return float(self.emission.max()) if self.K else 0.0

    @property
    def reflective(self) -> bool:  # src/scene.py:209-210
        return bool(self.K) and bool(np.any(self.albedo > 0.0))


def pack(scene) -> PackedScene:
    """Flatten any scene object exposing .surfaces/.medium/.bounds_min/.bounds_max."""
    dim = int(np.asarray(scene.bounds_min).size)
    k = dim  # vertices per primitive
    surfs = list(scene.surfaces)
    if surfs:
        verts = np.array([np.asarray(s.vertices, float) for s in surfs]).reshape(-1, k, dim)
        em = np.array([np.broadcast_to(np.asarray(s.emission, float), 3) for s in surfs])
        al = np.array([np.broadcast_to(np.asarray(s.albedo, float), 3) for s in surfs])
    else:
        verts = np.zeros((0, k, dim))
        em = np.zeros((0, 3))
        al = np.zeros((0, 3))
    return PackedScene(
        dim,
        verts,
        em,
        al,
        np.asarray(scene.bounds_min, float),
        np.asarray(scene.bounds_max, float),
        float(scene.medium.sigma_s),
        float(scene.medium.sigma_a),
        np.asarray(getattr(scene, "lights", np.zeros((0, 8))), float).reshape(-1, 8),
    )


def contains(ps: PackedScene, x) -> bool:  # src/scene.py:212-219
    eps = 1e-12 * ps.scale
    x = np.asarray(x, float)
    return bool(np.all((x >= ps.bmin - eps) & (x <= ps.bmax + eps)))


# ---------------------------------------------------------------------------
# Ray kernels (brute force, nearest hit, first-min tie break)
# ---------------------------------------------------------------------------


def _hits_2d(ps, o, d, t_eps):
    # src/scene.py:227-239 — cross-product segment test, inclusive 0 ≤ u ≤ 1.
    ao = ps.a[None] - o[:, None]
    e = ps.e1[None]
    den = d[:, None, 0] * e[:, :, 1] - d[:, None, 1] * e[:, :, 0]
    with np.errstate(divide="ignore", invalid="ignore"):
        t = (ao[:, :, 0] * e[:, :, 1] - ao[:, :, 1] * e[:, :, 0]) / den
        u = (ao[:, :, 0] * d[:, None, 1] - ao[:, :, 1] * d[:, None, 0]) / den
    ok = (np.abs(den) > 0.0) & (u >= 0.0) & (u <= 1.0) & (t > t_eps)
    return np.where(ok, t, np.inf)


def _hits_3d(ps, o, d, t_eps):
    # src/scene.py:242-268 — Möller–Trumbore, inclusive barycentrics.
    e1 = ps.e1[None]
    e2 = ps.e2[None]
    p = np.cross(d[:, None, :], e2)
    det = np.einsum("mkc,mkc->mk", np.broadcast_arrays(e1, p)[0], p)
    tv = o[:, None, :] - ps.a[None]
    with np.errstate(divide="ignore", invalid="ignore"):
        inv = 1.0 / det
        u = np.einsum("mkc,mkc->mk", tv, p) * inv
        q = np.cross(tv, e1)
        v = np.einsum("mkc,mkc->mk", np.broadcast_arrays(d[:, None, :], q)[0], q) * inv
        t = np.einsum("mkc,mkc->mk", np.broadcast_arrays(e2, q)[0], q) * inv
        ok = (
            np.isfinite(t)
            & (np.abs(det) > 0.0)
            & (u >= 0.0)
            & (v >= 0.0)
            & (u + v <= 1.0)
            & (t > t_eps)
        )
    return np.where(ok, t, np.inf)


_C_TRACE = {"lib": None, "threads": 0}


def use_c_trace(n_threads: int | None = None) -> bool:
    """Route `trace` through oracle/trace_c.c (same brute-force algorithm, OpenMP over rays).

    n_threads=0 switches back to numpy.  Returns whether the C helper is active.
    """
    import ctypes
    import os
    from pathlib import Path

    if n_threads == 0:
        _C_TRACE["threads"] = 0
        return False
    so = Path(__file__).resolve().parent / "_build" / "liboracle_trace.so"
    if not so.exists():
        from . import build_oracle

        build_oracle.build()
    if _C_TRACE["lib"] is None:
        L = ctypes.CDLL(str(so))
        L.oracle_trace.restype = None
        L.oracle_trace.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_void_p, ctypes.c_int64,
                                   ctypes.c_void_p, ctypes.c_void_p, ctypes.c_double, ctypes.c_void_p,
                                   ctypes.c_void_p, ctypes.c_int]
        _C_TRACE["lib"] = L
    _C_TRACE["threads"] = int(n_threads or len(os.sched_getaffinity(0)))
    return True


def _prim_array(ps: PackedScene) -> np.ndarray:
    if getattr(ps, "_prim", None) is None:
        if ps.dim == 3:
            ps._prim = np.ascontiguousarray(np.concatenate([ps.a, ps.e1, ps.e2], axis=1))
        else:
            ps._prim = np.ascontiguousarray(np.concatenate([ps.a, ps.e1], axis=1))
    return ps._prim


def trace(ps: PackedScene, origins, dirs, chunk: int = 4096):
    """Nearest hit per ray → (t, idx); misses (inf, −1).  src/scene.py:271-292.

    Rays are processed in chunks so the (m, K) temporaries stay bounded; every
    ray's result is independent of the chunking.
    """
    o = np.atleast_2d(np.asarray(origins, float))
    d = np.atleast_2d(np.asarray(dirs, float))
    m = o.shape[0]
    t_out = np.full(m, np.inf)
    i_out = np.full(m, -1, dtype=np.int64)
    if ps.K == 0 or m == 0:
        return t_out, i_out
    t_eps = T_EPS_REL * ps.scale
    if _C_TRACE["threads"]:
        P = _prim_array(ps)
        oc = np.ascontiguousarray(o)
        dc = np.ascontiguousarray(d)
        _C_TRACE["lib"].oracle_trace(ps.dim, ps.K, P.ctypes.data, m, oc.ctypes.data, dc.ctypes.data,
                                     t_eps, t_out.ctypes.data, i_out.ctypes.data, _C_TRACE["threads"])
        return t_out, i_out
    step = max(1, min(chunk, (1 << 22) // max(ps.K, 1)))
    kern = _hits_2d if ps.dim == 2 else _hits_3d
    for lo in range(0, m, step):
        sl = slice(lo, min(m, lo + step))
        tt = kern(ps, o[sl], d[sl], t_eps)
        j = np.argmin(tt, axis=1)
        best = tt[np.arange(tt.shape[0]), j]
        t_out[sl] = best
        i_out[sl] = np.where(np.isfinite(best), j, -1)
    return t_out, i_out


def bounds_exit(ps: PackedScene, origins, dirs):  # src/scene.py:295-303
    o = np.atleast_2d(origins)
    d = np.atleast_2d(dirs)
    with np.errstate(divide="ignore", invalid="ignore"):
        lo = (ps.bmin[None] - o) / d
        hi = (ps.bmax[None] - o) / d
    far = np.where(np.isnan(lo), np.inf, np.maximum(lo, hi))
    return np.min(far, axis=1)


def trace_or_bounds(ps, origins, dirs):  # src/scene.py:306-315
    t, idx = trace(ps, origins, dirs)
    tb = bounds_exit(ps, origins, dirs)
    return np.where(np.isfinite(t), t, tb), idx


def oriented_normals(ps, idx, dirs):  # src/scene.py:318-331
    dirs = np.atleast_2d(dirs)
    out = np.zeros_like(dirs)
    hit = idx >= 0
    if ps.K and np.any(hit):
        n = ps.normal[idx[hit]]
        sgn = np.sign(np.einsum("mc,mc->m", n, dirs[hit]))
        sgn = np.where(sgn == 0.0, 1.0, sgn)
        out[hit] = -n * sgn[:, None]
    return out


# ---------------------------------------------------------------------------
# Stratified directions + connectivity (src/scene.py:350-434)
# ---------------------------------------------------------------------------


def grid_shape_3d(n: int):  # src/scene.py:370-385
    target = math.sqrt(n / 2.0)
    best = None
    for rows in range(2, int(np.sqrt(n)) + 1):
        if n % rows or n // rows < 3:
            continue
        if best is None or abs(rows - target) < abs(best[0] - target):
            best = (rows, n // rows)
    if best is None:
        raise ValueError(f"n={n} is not expressible as rows x cols with rows >= 2 and cols >= 3")
    return best


def hull_adjacency(dirs):  # src/scene.py:388-399 (qhull, third party)
    from scipy.spatial import ConvexHull

    return np.asarray(ConvexHull(dirs, qhull_options="Qt").simplices, dtype=np.int64)


def directions(dim: int, n: int, rng, adjacency=None):
    """Jittered stratified directions; draws n (2D) or 2·rows·cols (3D) doubles.

    `adjacency` (E, 3) replaces the qhull connectivity when given (3D only);
    the draws are unchanged.  Returns (dirs, adjacency).
    """
    if dim == 2:
        if n < 3:
            raise ValueError("2D stratification needs n >= 3")
        xi = rng.random(n)
        th = (np.arange(n) + xi) * (2.0 * np.pi / n)
        d = np.column_stack([np.cos(th), np.sin(th)])
        k = np.arange(n)
        return d, np.column_stack([k, (k + 1) % n])
    rows, cols = grid_shape_3d(n)
    u = rng.random((rows, cols))
    v = rng.random((rows, cols))
    ri, ci = np.meshgrid(np.arange(rows), np.arange(cols), indexing="ij")
    z = 1.0 - 2.0 * (ri + u) / rows
    phi = (ci + v) * (2.0 * np.pi / cols)
    s = np.sqrt(np.clip(1.0 - z * z, 0.0, None))
    d = np.stack([s * np.cos(phi), s * np.sin(phi), z], axis=-1).reshape(-1, 3)
    adj = hull_adjacency(d) if adjacency is None else np.asarray(adjacency, np.int64)
    return d, adj


def uniform_dirs(dim: int, u):  # src/transport.py:274-285
    if dim == 2:
        th = 2.0 * np.pi * u
        return np.column_stack([np.cos(th), np.sin(th)])
    z = 1.0 - 2.0 * u[:, 0]
    phi = 2.0 * np.pi * u[:, 1]
    s = np.sqrt(np.clip(1.0 - z * z, 0.0, None))
    return np.column_stack([s * np.cos(phi), s * np.sin(phi), z])


# ---------------------------------------------------------------------------
# Surface shading (src/transport.py:127-254)
# ---------------------------------------------------------------------------


def emitter_quadrature(ps: PackedScene, n_per: int):
    """Midpoint samples per emitter → list of (points, weights, emission, normal)."""
    out = []
    for k in range(ps.K):
        if not np.any(ps.emission[k] > 0.0):
            continue
        V = ps.verts[k]
        if ps.dim == 2:
            a, b = V
            u = (np.arange(n_per) + 0.5) / n_per
            pts = a[None] + u[:, None] * (b - a)[None]
            length = float(np.linalg.norm(b - a))
            w = np.full(n_per, length / n_per)
            e = b - a
            nrm = np.array([-e[1], e[0]]) / length
        else:
            m = max(2, int(round(np.sqrt(n_per))))
            g = (np.arange(m) + 0.5) / m
            uu, vv = np.meshgrid(g, g, indexing="ij")
            uu, vv = uu.ravel().copy(), vv.ravel().copy()
            fold = uu + vv > 1.0
            uu[fold], vv[fold] = 1.0 - uu[fold], 1.0 - vv[fold]
            v0, v1, v2 = V
            pts = v0[None] + uu[:, None] * (v1 - v0)[None] + vv[:, None] * (v2 - v0)[None]
            cr = np.cross(v1 - v0, v2 - v0)
            area = 0.5 * float(np.linalg.norm(cr))
            w = np.full(m * m, area / (m * m))
            nrm = cr / np.linalg.norm(cr)
        out.append((pts, w, ps.emission[k], nrm))
    return out


def delta_incident(ps: PackedScene, org):
    """Extension (BASELINE.json cfg1/cfg2/cfg4 point lights, cfg3 directional light; the
    reference has area emitters only): per delta light the unit direction d toward
    it from each origin, its unoccluded attenuated geometric term and its rgb strength.
    Point light at P: r = |P − o|, term e^{−σt r} / max(r, 1e-6·scale)^{dim−1}, visible iff the
    nearest hit along d is at t ≥ r(1 − 1e-6) (the reference's shadow-ray rule,
    src/transport.py:213-214); r ≤ 1e-6·scale → 0.  Directional light: the ray must leave
    the scene without a hit (the light is outside the bounds), term e^{−σt s_b} with s_b the
    distance to the bounds exit along d (src/scene.py:295-303)."""
    org = np.atleast_2d(org)
    m, dim = org.shape
    off = 1e-6 * ps.scale
    out = []
    for row in ps.lights:
        kind, v, I = int(row[0]), row[1:1 + dim], row[4:7]
        val = np.zeros(m)
        if kind == 0:
            to = v[None] - org
            r = np.linalg.norm(to, axis=1)
            ok = r > off
            d = np.zeros_like(to)
            d[ok] = to[ok] / r[ok, None]
            if np.any(ok):
                th, _ = trace(ps, org[ok], d[ok])
                vis = th >= r[ok] * (1.0 - 1e-6)
                ii = np.flatnonzero(ok)[vis]
                val[ii] = np.exp(-ps.sigma_t * r[ii]) / np.maximum(r[ii], off) ** (dim - 1)
        else:
            d = np.broadcast_to(v, (m, dim)).copy()
            th, _ = trace(ps, org, d)
            vis = ~np.isfinite(th)
            if np.any(vis):
                val[vis] = np.exp(-ps.sigma_t * bounds_exit(ps, org[vis], d[vis]))
        out.append((d, val, I))
    return out


def delta_inscatter(ps: PackedScene, pts, g=0.0, toward=None):
    """Extension: mean incident radiance over the sphere (circle) at media points from the
    delta lights, Σ_l term_l·I_l / 4π (2π in 2D) — the quantity mean_surface_gather estimates
    for surfaces (src/transport.py:288-310).  g ≠ 0: each light is weighted 4π·p_g(d_l·toward),
    `toward` (m, 3) = the unit direction pointing AWAY from where the scattered light goes."""
    pts = np.atleast_2d(pts)
    out = np.zeros((pts.shape[0], 3))
    norm = 4.0 * np.pi if ps.dim == 3 else 2.0 * np.pi
    for d, val, I in delta_incident(ps, pts):
        w = val / norm
        if g != 0.0:
            w = w * (4.0 * np.pi * hg_phase(g, (d * toward).sum(axis=1)))
        out += w[:, None] * I[None]
    return out


def delta_single(ps: PackedScene, x):
    """Extension: the delta lights' own single scattering at the cache point x, in the units of
    the single moments (f̄ × mean incident radiance): value, gradient and Hessian of
    f̄·I·φ(x)/4π (2π in 2D) with the visibility V(x) held constant (a point visibility has no
    occlusion-aware derivative; the occlusion-aware terms of the method enter through the
    lit surfaces and media samples of the subdivision).  Point light: φ = e^{−σt r} r^{−k},
    k = dim − 1: φ′ = −(σt + k/r)φ, φ″ = ((σt + k/r)² + k/r²)φ, ∇φ = φ′u, Hφ = φ″uuᵀ + φ′/r(I − uuᵀ),
    u = (x − P)/r.  Directional light: φ = e^{−σt s_b}, s_b = (b_a − x_a)/d_a on the exit face a:
    ∇φ = σt φ e_a/d_a, Hφ = σt² φ e_a e_aᵀ/d_a²."""
    x = np.asarray(x, float)
    dim = x.size
    L, G, H = np.zeros(3), np.zeros((3, dim)), np.zeros((3, dim, dim))
    fbar = ps.sigma_s / (2.0 * np.pi if dim == 2 else 4.0 * np.pi)
    norm = 4.0 * np.pi if dim == 3 else 2.0 * np.pi
    sig, k = ps.sigma_t, dim - 1
    for row, (d, val, I) in zip(ps.lights, delta_incident(ps, x[None])):
        if not val[0] > 0.0:
            continue
        phi = val[0]
        if int(row[0]) == 0:
            w = x - row[1:1 + dim]
            r = float(np.linalg.norm(w))
            u = w / r
            a = sig + k / r
            d1 = -a * phi
            d2 = (a * a + k / (r * r)) * phi
            g = d1 * u
            h = d2 * np.outer(u, u) + d1 / r * (np.eye(dim) - np.outer(u, u))
        else:
            dv = d[0]
            with np.errstate(divide="ignore", invalid="ignore"):
                t = np.maximum((ps.bmin - x) / dv, (ps.bmax - x) / dv)
            t = np.where(np.isnan(t), np.inf, t)
            a = int(np.argmin(t))
            e = np.zeros(dim)
            e[a] = 1.0 / dv[a]
            g = sig * phi * e
            h = sig * sig * phi * np.outer(e, e)
        c = fbar / norm
        L += c * phi * I
        G += c * I[:, None] * g[None]
        H += c * I[:, None, None] * h[None]
    return L, G, H


def direct_light(ps: PackedScene, points, normals, n_light: int):
    """Shadow-ray quadrature of direct light; ÷π (3D) or ÷2 (2D).  src/transport.py:175-225."""
    points = np.atleast_2d(points)
    normals = np.atleast_2d(normals)
    m = points.shape[0]
    acc = np.zeros((m, 3))
    quad = emitter_quadrature(ps, n_light)
    if not quad and not len(ps.lights):
        return acc
    off = 1e-6 * ps.scale
    org = points + off * normals
    for d, val, I in delta_incident(ps, org):  # extension: delta lights, same cosine and ÷π / ÷2
        cp = np.clip(np.einsum("md,md->m", normals, d), 0.0, None)
        acc += (cp * val)[:, None] * I[None]
    for pts, wts, E, N in quad:
        for j in range(pts.shape[0]):
            to = pts[j][None] - org
            r = np.linalg.norm(to, axis=1)
            ok = r > off
            d = np.zeros_like(to)
            d[ok] = to[ok] / r[ok, None]
            cp = np.clip(np.einsum("md,md->m", normals, d), 0.0, None)
            cq = np.abs(d @ N)
            live = ok & (cp > 0.0) & (cq > 0.0)
            if not np.any(live):
                continue
            th, _ = trace(ps, org[live], d[live])
            vis = th >= r[live] * (1.0 - 1e-6)
            g = np.zeros(m)
            ii = np.flatnonzero(live)[vis]
            g[ii] = (
                cp[ii] * cq[ii] / np.maximum(r[ii], off) ** (ps.dim - 1)
                * np.exp(-ps.sigma_t * r[ii]) * wts[j]
            )
            acc += g[:, None] * E[None]
    return acc / (np.pi if ps.dim == 3 else 2.0)


def surface_radiance(ps: PackedScene, idx, points, dirs, n_light: int):
    """Emission + albedo·direct at hits; bounds terminations → 0.  src/transport.py:228-254."""
    idx = np.asarray(idx)
    out = np.zeros((idx.size, 3))
    hit = idx >= 0
    if not np.any(hit):
        return out
    out[hit] = ps.emission[idx[hit]]
    if ps.reflective:
        needs = np.any(ps.albedo[idx[hit]] > 0.0, axis=1)
        if np.any(needs):
            sub = np.flatnonzero(hit)[needs]
            nrm = oriented_normals(ps, idx[sub], dirs[sub])
            out[sub] += ps.albedo[idx[sub]] * direct_light(ps, points[sub], nrm, n_light)
    return out


def gather_mean(ps, points, dirs_pp, n_light):  # src/transport.py:288-310
    m, n, dim = dirs_pp.shape
    org = np.repeat(points, n, axis=0)
    dd = dirs_pp.reshape(-1, dim)
    tot = np.zeros((m * n, 3))
    for lo in range(0, m * n, CHUNK):
        sl = slice(lo, min(lo + CHUNK, m * n))
        s, idx = trace_or_bounds(ps, org[sl], dd[sl])
        lo_r = surface_radiance(ps, idx, org[sl] + s[:, None] * dd[sl], dd[sl], n_light)
        tot[sl] = np.exp(-ps.sigma_t * s)[:, None] * lo_r
    return tot.reshape(m, n, 3).mean(axis=1)


def hg_phase(g, c):
    """Henyey–Greenstein phase p(cos θ), normalised over the sphere (extension)."""
    return (1.0 - g * g) / (4.0 * np.pi * (1.0 + g * g - 2.0 * g * c) ** 1.5)


def hg_sample(g, cur, u0, u1):
    """Extension: a direction about the unit vectors `cur` (m, 3) with cos θ ~ HG(g) (g ≠ 0)
    from u0 and azimuth 2π·u1, in the branchless orthonormal basis of Duff et al. (2017)."""
    s = (1.0 - g * g) / (1.0 - g + 2.0 * g * u0)
    ct = (1.0 + g * g - s * s) / (2.0 * g)
    st = np.sqrt(np.maximum(0.0, 1.0 - ct * ct))
    phi = 2.0 * np.pi * u1
    x, y, z = cur[:, 0], cur[:, 1], cur[:, 2]
    sign = np.copysign(1.0, z)
    a = -1.0 / (sign + z)
    b = x * y * a
    t1 = np.stack([1.0 + sign * x * x * a, sign * b, -sign * x], axis=1)
    t2 = np.stack([b, sign + y * y * a, -y], axis=1)
    return (st * np.cos(phi))[:, None] * t1 + (st * np.sin(phi))[:, None] * t2 + ct[:, None] * cur


def gather_mean_bounces(ps, points, dirs_pp, n_light, extras, bounces, g=0.0, x=None):
    """Extension (BASELINE.json cfg3 "multiple scattering up to 4 bounces"; the reference
    stops at one extra bounce): the media-sample gather continued by up to `bounces` − 1
    further media scattering events per gather path, restating the multiple-scattering loop
    of path_trace_radiance (src/transport.py:362-388) — collision distance
    −log1p(−u)/σt against the current segment, weight σs/σt per collision, a uniform new
    direction, T·L_o at its surface hit added with the path weight.  `extras` (m, n, B−1, d')
    holds per path and bounce (u_dist, direction draws): the record's PCG64 stream continued
    after every draw the reference makes (build_record).  bounces = 1 → gather_mean.

    Extension g ≠ 0 (3D; BASELINE cfg2/cfg3's Henyey–Greenstein media): scattering at the media
    sample y toward the cache point x weighs each gather path by 4π·p_g(ω·w), w = (y − x)/|y − x|
    (light arriving along −ω leaves toward x), and every further media event samples its new
    direction from HG(g) about the current one (hg_sample; the σs/σt weight is unchanged)."""
    m, n, dim = dirs_pp.shape
    org = np.repeat(points, n, axis=0)
    dd = dirs_pp.reshape(-1, dim)
    s, idx = trace_or_bounds(ps, org, dd)
    tot = np.exp(-ps.sigma_t * s)[:, None] * surface_radiance(ps, idx, org + s[:, None] * dd, dd, n_light)
    w0 = np.ones(m * n)
    if g != 0.0:
        dx = org - np.asarray(x, float)[None]
        wk = dx / np.sqrt((dx * dx).sum(axis=1))[:, None]
        w0 = 4.0 * np.pi * hg_phase(g, (dd * wk).sum(axis=1))
        tot = tot * w0[:, None]
    if bounces > 1 and ps.sigma_t > 0.0:
        ex = extras.reshape(m * n, bounces - 1, -1)
        w = w0.copy()
        alive = np.ones(m * n, bool)
        pos, cur_d, cur_s = org, dd, s
        for b in range(bounces - 1):
            t = -np.log1p(-ex[:, b, 0]) / ps.sigma_t
            col = alive & (t < cur_s)
            if not np.any(col):
                break
            pos = pos + np.where(col, t, 0.0)[:, None] * cur_d
            w = w * np.where(col, ps.sigma_s / ps.sigma_t, 1.0)
            if g != 0.0:
                nd = hg_sample(g, cur_d, ex[:, b, 1], ex[:, b, 2])
            else:
                nd = uniform_dirs(dim, ex[:, b, 1] if dim == 2 else ex[:, b, 1:3])
            s2 = np.zeros(m * n)
            s2[col], idx2 = trace_or_bounds(ps, pos[col], nd[col])
            lo2 = surface_radiance(ps, idx2, pos[col] + s2[col, None] * nd[col], nd[col], n_light)
            tot[col] += w[col, None] * np.exp(-ps.sigma_t * s2[col])[:, None] * lo2
            if len(ps.lights):  # extension: the delta lights scattered at this collision toward −cur_d
                tot[col] += w[col, None] * delta_inscatter(ps, pos[col], g, cur_d[col])
            alive = col
            cur_d = nd
            cur_s = s2
    return tot.reshape(m, n, 3).mean(axis=1)


# ---------------------------------------------------------------------------
# Form factors with derivatives (src/formfactor.py:85-343)
# ---------------------------------------------------------------------------


def segment_ff(x, y0, y1):
    """2D segment F = γ/2π with ∇F, HF (Appendix-B chain).  src/formfactor.py:85-158."""
    u = y0 - x
    v = y1 - x
    r0 = np.linalg.norm(u, axis=1)
    r1 = np.linalg.norm(v, axis=1)
    ok = (r0 > 0.0) & (r1 > 0.0)
    a = np.where(ok, r0, 1.0)
    b = np.where(ok, r1, 1.0)
    dot = np.einsum("md,md->m", u, v)
    crs = u[:, 0] * v[:, 1] - u[:, 1] * v[:, 0]
    g = np.arctan2(np.abs(crs), dot)
    ok &= (g > GAMMA_MIN) & (g < np.pi - GAMMA_MIN)
    val = np.where(ok, g / (2.0 * np.pi), 0.0)
    c = np.clip(dot / (a * b), -1.0, 1.0)
    sn = np.where(ok, np.abs(crs) / (a * b), 1.0)
    gc = (c / a**2)[:, None] * u + (c / b**2)[:, None] * v - (u + v) / (a * b)[:, None]
    grad = -(gc / sn[:, None]) / (2.0 * np.pi)
    I = np.eye(2)[None]
    uu = u[:, :, None] * u[:, None, :]
    vv = v[:, :, None] * v[:, None, :]
    jc = (
        u[:, :, None] * gc[:, None, :] / (a**2)[:, None, None]
        + 2.0 * (c / a**4)[:, None, None] * uu
        - (c / a**2)[:, None, None] * I
        + v[:, :, None] * gc[:, None, :] / (b**2)[:, None, None]
        + 2.0 * (c / b**4)[:, None, None] * vv
        - (c / b**2)[:, None, None] * I
        + 2.0 * I / (a * b)[:, None, None]
        - (u + v)[:, :, None] * (u / (a**3 * b)[:, None] + v / (a * b**3)[:, None])[:, None, :]
    )
    hess = -(jc / sn[:, None, None] + (c / sn**3)[:, None, None] * (gc[:, :, None] * gc[:, None, :])) / (2.0 * np.pi)
    grad = np.where(ok[:, None], grad, 0.0)
    hess = np.where(ok[:, None, None], hess, 0.0)
    return ok, val, grad, 0.5 * (hess + np.swapaxes(hess, 1, 2))


def triangle_ff(x, y1, y2, y3):
    """3D triangle F = Ω/4π, Ω = 2·atan2(|A|, B), with ∇F, HF.  src/formfactor.py:182-343."""
    R = [y1 - x, y2 - x, y3 - x]
    rr = [np.linalg.norm(w, axis=1) for w in R]
    pos = (rr[0] > 0.0) & (rr[1] > 0.0) & (rr[2] > 0.0)
    r = [np.where(pos, q, 1.0) for q in rr]
    A = np.einsum("md,md->m", R[0], np.cross(R[1], R[2]))
    d12 = np.einsum("md,md->m", R[0], R[1])
    d23 = np.einsum("md,md->m", R[1], R[2])
    d13 = np.einsum("md,md->m", R[0], R[2])
    B = r[0] * r[1] * r[2] + d12 * r[2] + d23 * r[0] + d13 * r[1]
    gA = -(np.cross(R[0], R[1]) + np.cross(R[1], R[2]) + np.cross(R[2], R[0]))
    gr = [-R[i] / r[i][:, None] for i in range(3)]
    gB = (
        (r[1] * r[2])[:, None] * gr[0] + (r[0] * r[2])[:, None] * gr[1] + (r[0] * r[1])[:, None] * gr[2]
        + d12[:, None] * gr[2] - r[2][:, None] * (R[0] + R[1])
        + d23[:, None] * gr[0] - r[0][:, None] * (R[1] + R[2])
        + d13[:, None] * gr[1] - r[1][:, None] * (R[0] + R[2])
    )
    I = np.eye(3)[None]

    def ob(p, q):
        return p[:, :, None] * q[:, None, :]

    Jr = [(I - ob(R[i], R[i]) / (r[i] ** 2)[:, None, None]) / r[i][:, None, None] for i in range(3)]
    g12 = r[1][:, None] * gr[0] + r[0][:, None] * gr[1]
    g23 = r[2][:, None] * gr[1] + r[1][:, None] * gr[2]
    g13 = r[2][:, None] * gr[0] + r[0][:, None] * gr[2]
    HB = (
        (r[1] * r[2])[:, None, None] * Jr[0] + (r[0] * r[2])[:, None, None] * Jr[1]
        + (r[0] * r[1])[:, None, None] * Jr[2]
        + ob(gr[0], g23) + ob(gr[1], g13) + ob(gr[2], g12)
    )
    for dij, k, p, q in ((d12, 2, R[0], R[1]), (d23, 0, R[1], R[2]), (d13, 1, R[0], R[2])):
        HB = HB + dij[:, None, None] * Jr[k] + 2.0 * r[k][:, None, None] * I - ob(gr[k], p + q) - ob(p + q, gr[k])
    aA = np.abs(A)
    ok = pos & (aA >= A_REL_MIN * r[0] * r[1] * r[2])
    val = np.where(pos & ((aA > 0.0) | (B > 0.0)), 2.0 * np.arctan2(aA, B) / (4.0 * np.pi), 0.0)
    sg = np.where(A >= 0.0, 1.0, -1.0)
    gU = sg[:, None] * gA
    den = np.where(ok, A * A + B * B, 1.0)
    num = B[:, None] * gU - aA[:, None] * gB
    grad = num / den[:, None] / (2.0 * np.pi)
    gD = 2.0 * aA[:, None] * gU + 2.0 * B[:, None] * gB
    hess = (
        (ob(gU, gB) - ob(gB, gU) - aA[:, None, None] * HB) / den[:, None, None]
        - ob(num, gD) / (den**2)[:, None, None]
    ) / (2.0 * np.pi)
    grad = np.where(ok[:, None], grad, 0.0)
    hess = np.where(ok[:, None, None], hess, 0.0)
    val = np.where(ok | (pos & (B > 0.0)), val, 0.0)
    return ok, val, grad, 0.5 * (hess + np.swapaxes(hess, 1, 2))


# ---------------------------------------------------------------------------
# Record build: subdivision + moment assembly (src/subdivision.py:136-393)
# ---------------------------------------------------------------------------


@dataclass
class RecordBuild:
    """Everything the GPU path exposes per record, for element-level checks."""

    dirs: np.ndarray
    adjacency: np.ndarray
    s: np.ndarray
    idx: np.ndarray
    surface_radiance: np.ndarray
    ring_radii: np.ndarray
    counts: np.ndarray  # live rings per direction
    media_radiance: np.ndarray  # (P, 3) in (direction, ring) row-major order
    L: np.ndarray  # (2, 3) single, multiple
    grad: np.ndarray  # (2, 3, dim)
    hess: np.ndarray  # (2, 3, dim, dim)
    stats: dict


def build_record(
    ps: PackedScene,
    x,
    n_angular: int | None = None,
    march_step: float = 0.1,
    rng_seed=None,
    n_inner: int = 1,
    n_light_samples: int = 16,
    adjacency=None,
    media_bounces: int = 1,
    hg_g: float = 0.0,
) -> RecordBuild:
    """One cache point: `estimate_moments` (src/subdivision.py:373-393) in one pass.

    Follows build_subdivision (:136-234), _make_ring (:237-253) and
    assemble_moments (:287-370): per ring, elements whose representative
    (first-argmax-distance) vertex carries positive radiance are evaluated;
    degenerate ones are dropped; weights f̄·step (media → multiple) and f̄
    (surface → single).
    """
    x = np.asarray(x, float)
    dim = x.size
    if march_step <= 0.0:
        raise ValueError("march_step must be positive")
    if not contains(ps, x):
        raise ValueError("subdivision center lies outside the medium bounds")
    n = n_angular if n_angular is not None else {2: 256, 3: 16384}[dim]
    rng = np.random.default_rng(rng_seed)
    dirs, adj = directions(dim, n, rng, adjacency)

    org = np.broadcast_to(x, (n, dim)).copy()
    s, idx = trace_or_bounds(ps, org, dirs)
    hit_pts = org + s[:, None] * dirs
    lo_surf = surface_radiance(ps, idx, hit_pts, dirs, n_light_samples)

    R = int(np.floor(float(np.max(s)) / march_step + 0.5))
    radii = (np.arange(1, R + 1) - 0.5) * march_step
    live = radii[None, :] < s[:, None]
    counts = live.sum(axis=1)
    media_pts = org[:, None, :] + radii[None, :, None] * dirs[:, None, :]
    media_rad = np.zeros((n, R, 3))
    flat = np.flatnonzero(live)
    if flat.size and ps.sigma_s > 0.0:
        p = media_pts.reshape(-1, dim)[flat]
        if dim == 2:
            u = rng.random((p.shape[0], n_inner))
            gd = uniform_dirs(2, u.reshape(-1)).reshape(p.shape[0], n_inner, 2)
        else:
            u = rng.random((p.shape[0], n_inner, 2))
            gd = uniform_dirs(3, u.reshape(-1, 2)).reshape(p.shape[0], n_inner, 3)
        if media_bounces > 1 or hg_g != 0.0:  # extension: the stream continues after the reference's draws
            ex = rng.random((p.shape[0], n_inner, media_bounces - 1, 2 if dim == 2 else 3))
            media_rad.reshape(-1, 3)[flat] = ps.sigma_s * gather_mean_bounces(ps, p, gd, n_light_samples, ex,
                                                                            media_bounces, hg_g, x)
        else:
            media_rad.reshape(-1, 3)[flat] = ps.sigma_s * gather_mean(ps, p, gd, n_light_samples)
        if len(ps.lights):  # extension: the delta lights' in-scatter at every media sample
            dx = p - x[None]
            wk = dx / np.sqrt((dx * dx).sum(axis=1))[:, None]
            media_rad.reshape(-1, 3)[flat] += ps.sigma_s * delta_inscatter(ps, p, hg_g, wk)

    fbar = ps.sigma_s / (2.0 * np.pi if dim == 2 else 4.0 * np.pi)
    sig = ps.sigma_t
    acc_L = np.zeros((2, 3))
    acc_g = np.zeros((2, 3, dim))
    acc_h = np.zeros((2, 3, dim, dim))
    n_eval = 0
    n_drop = 0
    stars = 0
    is_hit = idx >= 0

    def ring(kind, pts, rad, dist, weight):
        nonlocal n_eval, n_drop
        V = pts[adj]
        Dv = dist[adj]
        rep = np.argmax(Dv, axis=1)
        e = np.arange(adj.shape[0])
        r_rad = rad[adj][e, rep]
        keep = np.any(r_rad > 0.0, axis=1)
        if not np.any(keep):
            return
        V = V[keep]
        r_rad = r_rad[keep]
        rp = V[np.arange(V.shape[0]), rep[keep]]
        rd = Dv[keep][np.arange(V.shape[0]), rep[keep]]
        if dim == 2:
            ok, F, gF, HF = segment_ff(x[None], V[:, 0], V[:, 1])
        else:
            ok, F, gF, HF = triangle_ff(x[None], V[:, 0], V[:, 1], V[:, 2])
        n_eval += int(keep.sum())
        n_drop += int((~ok).sum())
        if not np.any(ok):
            return
        F, gF, HF, r_rad, rp, rd = F[ok], gF[ok], HF[ok], r_rad[ok], rp[ok], rd[ok]
        w = x[None] - rp
        T = np.exp(-sig * rd)
        gT = -sig * w / rd[:, None] * T[:, None]  # src/transport.py:108-110
        ww = w[:, :, None] * w[:, None, :]
        HT = -sig * (
            np.eye(dim)[None] / rd[:, None, None] - ww / (rd**3)[:, None, None]
            - sig * ww / (rd**2)[:, None, None]
        ) * T[:, None, None]  # src/transport.py:113-119
        val = T * F
        ge = T[:, None] * gF + gT * F[:, None]
        he = (
            T[:, None, None] * HF + gT[:, :, None] * gF[:, None, :]
            + gF[:, :, None] * gT[:, None, :] + HT * F[:, None, None]
        )
        kk = 0 if kind == "surface" else 1
        wt = fbar * weight
        acc_L[kk] += wt * np.einsum("e,ec->c", val, r_rad)
        acc_g[kk] += wt * np.einsum("ed,ec->cd", ge, r_rad)
        acc_h[kk] += wt * np.einsum("edf,ec->cdf", he, r_rad)

    for i in range(R):
        lv = live[:, i]
        if not np.any(lv):
            continue
        pts = np.where(lv[:, None], media_pts[:, i, :], hit_pts)
        rad = np.where(lv[:, None], media_rad[:, i, :], 0.0)
        dist = np.where(lv, radii[i], s)
        stars += int((~lv & is_hit)[adj].sum())
        ring("media", pts, rad, dist, march_step)
    ring("surface", hit_pts, lo_surf, s, 1.0)

    acc_h = 0.5 * (acc_h + np.swapaxes(acc_h, -1, -2))
    if len(ps.lights):  # extension: the delta lights' single scattering at x itself
        dL, dG, dH = delta_single(ps, x)
        acc_L[0] += dL
        acc_g[0] += dG
        acc_h[0] += dH
    stats = {
        "elements_evaluated": n_eval,
        "elements_dropped": n_drop,
        "dropped_fraction": (n_drop / n_eval) if n_eval else 0.0,
        "star_vertices": stars,
    }
    return RecordBuild(
        dirs=dirs,
        adjacency=adj,
        s=s,
        idx=idx,
        surface_radiance=lo_surf,
        ring_radii=radii,
        counts=counts,
        media_radiance=media_rad.reshape(-1, 3)[flat] if flat.size else np.zeros((0, 3)),
        L=acc_L,
        grad=acc_g,
        hess=acc_h,
        stats=stats,
    )


# ---------------------------------------------------------------------------
# Records: luminance Hessian → eigen → radii (src/cache.py:59-189, src/numerics.py)
# ---------------------------------------------------------------------------


def _sorted_eig(vals, vecs):  # src/numerics.py:51-53
    o = np.argsort(-np.abs(vals), kind="stable")
    return vals[o].copy(), vecs[:, o].copy()


def eig2(m):  # src/numerics.py:56-73
    a, b, c = m[0, 0], m[0, 1], m[1, 1]
    mean, hd = 0.5 * (a + c), 0.5 * (a - c)
    disc = np.hypot(hd, b)
    l1, l2 = mean + disc, mean - disc
    if disc <= 1e-14 * max(abs(mean), 1e-300):
        V = np.eye(2)
    else:
        v = np.array([hd + disc, b])
        alt = np.array([b, -hd + disc])
        if alt @ alt > v @ v:
            v = alt
        v = v / np.linalg.norm(v)
        V = np.column_stack([v, [-v[1], v[0]]])
    return _sorted_eig(np.array([l1, l2]), V)


def eig3(m):  # src/numerics.py:76-124, analytic with None on degeneracy
    sc = np.max(np.abs(m))
    if sc == 0.0:
        return np.zeros(3), np.eye(3)
    p1 = m[0, 1] ** 2 + m[0, 2] ** 2 + m[1, 2] ** 2
    if p1 <= (1e-14 * sc) ** 2:
        return _sorted_eig(np.diagonal(m).copy(), np.eye(3))
    q = np.trace(m) / 3.0
    p2 = (m[0, 0] - q) ** 2 + (m[1, 1] - q) ** 2 + (m[2, 2] - q) ** 2 + 2.0 * p1
    p = np.sqrt(p2 / 6.0)
    Bm = (m - q * np.eye(3)) / p
    r = np.clip(np.linalg.det(Bm) / 2.0, -1.0, 1.0)
    phi = np.arccos(r) / 3.0
    hi = q + 2.0 * p * np.cos(phi)
    lo = q + 2.0 * p * np.cos(phi + 2.0 * np.pi / 3.0)
    vals = np.array([hi, 3.0 * q - hi - lo, lo])
    if min(abs(vals[0] - vals[1]), abs(vals[1] - vals[2]), abs(vals[0] - vals[2])) < 1e-6 * sc:
        return None
    V = np.empty((3, 3))
    for k, lam in enumerate(vals):
        A = m - lam * np.eye(3)
        cs = [np.cross(A[0], A[1]), np.cross(A[0], A[2]), np.cross(A[1], A[2])]
        v = cs[int(np.argmax([c @ c for c in cs]))]
        nv = np.linalg.norm(v)
        if nv < 1e-12 * sc * sc:
            return None
        V[:, k] = v / nv
    return _sorted_eig(vals, V)


def eigen_sym(m):  # src/numerics.py:127-166
    m = 0.5 * (m + m.T)
    sc = float(np.max(np.abs(m)))
    d = m.shape[0]
    if sc == 0.0:
        return np.zeros(d), np.eye(d)
    mu = m / sc
    if d == 2:
        vals, V = eig2(mu)
    else:
        res = eig3(mu)
        if res is not None:
            vals, V = res
            recon = (V * vals) @ V.T
            if (np.linalg.norm(recon - mu) > 0.5e-6 * np.linalg.norm(mu)
                    or np.linalg.norm(V.T @ V - np.eye(3)) > 1e-10):
                res = None
        if res is None:
            w, Q = np.linalg.eigh(mu)
            vals, V = _sorted_eig(w, Q)
    return vals * sc, V


def valid_radii(L, lam, eps, dim, scale):  # src/cache.py:59-91
    lam = np.abs(np.asarray(lam, float))
    rmax = R_MAX_FRACTION * scale
    floor = CURVATURE_FLOOR * L / scale**2
    out = np.full(dim, rmax)
    lv = lam > floor
    if np.any(lv):
        if dim == 2:
            out[lv] = (4.0 * L * eps / (np.pi * lam[lv])) ** 0.25
        else:
            out[lv] = (15.0 * L * eps / (4.0 * np.pi * lam[lv])) ** 0.2
    return np.minimum(out, rmax)


@dataclass(frozen=True)
class Record:
    position: np.ndarray
    value: np.ndarray
    grad: np.ndarray
    axes: np.ndarray
    radii: np.ndarray

    def support(self, x):  # src/cache.py:112-116
        along = (np.asarray(x, float) - self.position) @ self.axes
        return 1.0 - float(np.sqrt(np.sum((along / self.radii) ** 2)))

    def extrapolate(self, x):  # src/cache.py:118-121
        return np.clip(self.value + self.grad @ (np.asarray(x, float) - self.position), 0.0, None)


def make_record(x, L, grad, hess, epsilon, scale, max_emission, anisotropic=True) -> Record:
    """src/cache.py:146-189."""
    x = np.asarray(x, float)
    dim = x.size
    lum = max(float(L @ LUMA), L_FLOOR_FRACTION * max_emission)
    H = np.einsum("cij,c->ij", hess, LUMA)
    if lum <= 0.0:
        axes, radii = np.eye(dim), np.full(dim, R_MAX_FRACTION * scale)
    else:
        vals, axes = eigen_sym(H)
        if not anisotropic:
            vals = np.full(dim, np.max(np.abs(vals)))
        radii = valid_radii(lum, vals, epsilon, dim, scale)
    return Record(x, np.array(L, float).copy(), np.array(grad, float).copy(), axes, radii)


# ---------------------------------------------------------------------------
# Cache index + interpolation (src/cache.py:235-360)
# ---------------------------------------------------------------------------


def weight_cubic(d):  # src/cache.py:49-56
    d = min(max(float(d), 0.0), 1.0)
    return 3.0 * d * d - 2.0 * d * d * d


class Cache:
    """Linear-scan cache: the reference tree query returns exactly this set (src/cache.py:317-334)."""

    def __init__(self, records=()):
        self.records = list(records)

    def query(self, x):
        return [r for r in self.records if r.support(x) > 0.0]


def interpolate(cache: Cache, x):  # src/cache.py:342-360
    recs = cache.query(x)
    if not recs:
        return None
    num = np.zeros(3)
    den = 0.0
    for r in recs:
        w = weight_cubic(r.support(x))
        num += w * r.extrapolate(x)
        den += w
    return None if den <= 0.0 else num / den


# ---------------------------------------------------------------------------
# Camera march with a frozen cache pair (src/renderer.py:133-193, :335-484)
# ---------------------------------------------------------------------------


def seed_seq(*parts):  # src/renderer.py:278-279
    return np.random.SeedSequence([int(p) & 0xFFFFFFFF for p in parts])


def camera_basis(position, look_at, up):  # src/renderer.py:158-170
    f = np.asarray(look_at, float) - np.asarray(position, float)
    f = f / np.linalg.norm(f)
    r = np.cross(f, np.asarray(up, float))
    r = r / np.linalg.norm(r)
    return f, r, np.cross(r, f)


def camera_rays(position, look_at, up, fov, w, h, jitter):  # src/renderer.py:172-193
    f, r, u_ = camera_basis(position, look_at, up)
    th = np.tan(np.radians(fov) * 0.5)
    px, py = np.meshgrid(np.arange(w), np.arange(h))
    u = (px + jitter[..., 0]) / w
    v = (py + jitter[..., 1]) / h
    xn = (2.0 * u - 1.0) * th * (w / h)
    yn = (1.0 - 2.0 * v) * th
    d = f[None, None] + xn[..., None] * r[None, None] + yn[..., None] * u_[None, None]
    d = d / np.linalg.norm(d, axis=-1, keepdims=True)
    o = np.broadcast_to(np.asarray(position, float), d.shape).reshape(-1, 3).copy()
    return o, d.reshape(-1, 3)


def bounds_span(ps, o, d):  # src/renderer.py:382-394
    with np.errstate(divide="ignore", invalid="ignore"):
        t1 = (ps.bmin[None] - o) / d
        t2 = (ps.bmax[None] - o) / d
    near = np.where(np.isnan(np.minimum(t1, t2)), -np.inf, np.minimum(t1, t2))
    far = np.where(np.isnan(np.maximum(t1, t2)), np.inf, np.maximum(t1, t2))
    t_in = np.clip(near.max(axis=1), 0.0, None)
    t_out = far.min(axis=1)
    return t_in, t_out, t_out > t_in


@dataclass
class RenderParams:
    epsilon: float = 0.05
    spp: int = 1
    march_step: float = 0.1
    n_angular: int | None = None
    seed: int = 0
    n_light_samples: int = 16
    n_inner: int = 1
    anisotropic: bool = True


def point_value(ps, y, single: Cache, multiple: Cache, prm: RenderParams, seed, stats, adjacency_fn=None,
                frozen=True):
    """Shading value at a march point (src/renderer.py:335-368); frozen=False inserts."""
    a = interpolate(single, y)
    b = interpolate(multiple, y)
    if a is not None and b is not None:
        stats["cache_hits"] += 1
        return a + b
    stats["direct_evaluations"] += 1
    if not frozen:
        value, (rs, rm) = compute_pair(ps, y, prm, seed, adjacency_fn)
        if a is None:
            single.records.append(rs)
        if b is None:
            multiple.records.append(rm)
        a2, b2 = interpolate(single, y), interpolate(multiple, y)
        return a2 + b2 if (a2 is not None and b2 is not None) else value
    rb = build_record(
        ps, y, n_angular=prm.n_angular, march_step=prm.march_step, rng_seed=seed,
        n_inner=prm.n_inner, n_light_samples=prm.n_light_samples,
        adjacency=None if adjacency_fn is None else adjacency_fn(seed),
    )
    return rb.L[0] + rb.L[1]


def render_camera(ps, cam: dict, single: Cache, multiple: Cache, prm: RenderParams,
                  pixels=None, adjacency_fn=None, frozen=True):
    """Frozen-cache camera image (src/renderer.py:440-484); `pixels` restricts to a crop.

    `cam` = {position, look_at, up, fov, width, height}.  Returns (image (h·w, 3), stats).
    """
    h, w = cam["height"], cam["width"]
    sig = ps.sigma_t
    rng = np.random.default_rng(seed_seq(prm.seed, 101))
    img = np.zeros((h * w, 3))
    stats = {"cache_hits": 0, "direct_evaluations": 0}
    pix = np.arange(h * w) if pixels is None else np.asarray(pixels)
    for k in range(prm.spp):
        jit = rng.random((h, w, 2)) if prm.spp > 1 else np.full((h, w, 2), 0.5)
        o, d = camera_rays(cam["position"], cam["look_at"], cam["up"], cam["fov"], w, h, jit)
        t_s, idx = trace(ps, o[pix], d[pix])
        hp = o[pix] + np.where(np.isfinite(t_s), t_s, 0.0)[:, None] * d[pix]
        lo = surface_radiance(ps, idx, hp, d[pix], prm.n_light_samples)
        t_in, t_out, valid = bounds_span(ps, o[pix], d[pix])
        t_end = np.minimum(t_s, t_out)
        for q, i in enumerate(pix):
            if not valid[q]:
                if idx[q] >= 0:
                    img[i] += lo[q]
                continue
            steps = int(np.floor((t_end[q] - t_in[q]) / prm.march_step + 0.5))
            acc = np.zeros(3)
            for m in range(1, steps + 1):
                tk = t_in[q] + (m - 0.5) * prm.march_step
                y = o[i] + tk * d[i]
                J = point_value(ps, y, single, multiple, prm, seed_seq(prm.seed, 211, k, i, m), stats, adjacency_fn,
                                frozen)
                acc += np.exp(-sig * (tk - t_in[q])) * (4.0 * np.pi) * J * prm.march_step
            if idx[q] >= 0:
                acc += np.exp(-sig * max(0.0, t_end[q] - t_in[q])) * lo[q]
            img[i] += acc
    return img / prm.spp, stats


# ---------------------------------------------------------------------------
# Cache population and field render (src/renderer.py:282-327, :335-368, :425-437)
# ---------------------------------------------------------------------------


def march_points(ps, target: dict, march_step: float):
    """Scanline march points (src/renderer.py:282-299).

    `target` = {"kind": "field", nx, ny, bmin, bmax} or {"kind": "camera", position,
    look_at, up, fov, width, height}.
    """
    if target["kind"] == "field":
        nx, ny = target["nx"], target["ny"]
        lo, hi = np.asarray(target["bmin"], float), np.asarray(target["bmax"], float)
        dx = (hi[0] - lo[0]) / nx
        dy = (hi[1] - lo[1]) / ny
        for iy in range(ny):
            for ix in range(nx):
                yield np.array([lo[0] + (ix + 0.5) * dx, hi[1] - (iy + 0.5) * dy])
        return
    h, w = target["height"], target["width"]
    o, d = camera_rays(target["position"], target["look_at"], target["up"], target["fov"], w, h,
                       np.full((h, w, 2), 0.5))
    t_s, _ = trace(ps, o, d)
    t_in, t_out, valid = bounds_span(ps, o, d)
    t_end = np.minimum(t_s, t_out)
    for i in range(o.shape[0]):
        if not valid[i]:
            continue
        n_steps = int(np.floor((t_end[i] - t_in[i]) / march_step + 0.5))
        for k in range(1, n_steps + 1):
            yield o[i] + (t_in[i] + (k - 0.5) * march_step) * d[i]


def compute_pair(ps, x, prm: RenderParams, seed, adjacency_fn=None):
    """CacheSet.compute (src/renderer.py:231-262) for the ours-* modes → (J, (rec_s, rec_m))."""
    rb = build_record(ps, x, n_angular=prm.n_angular, march_step=prm.march_step, rng_seed=seed,
                      n_inner=prm.n_inner, n_light_samples=prm.n_light_samples,
                      adjacency=None if adjacency_fn is None else adjacency_fn(seed))
    recs = tuple(make_record(x, rb.L[k], rb.grad[k], rb.hess[k], prm.epsilon, ps.scale, ps.max_emission,
                             anisotropic=prm.anisotropic) for k in (0, 1))
    return rb.L[0] + rb.L[1], recs


def populate_cache(ps, target: dict, prm: RenderParams, adjacency_fn=None):
    """Sequential greedy insertion (src/renderer.py:302-327) → (single, multiple, points)."""
    single, multiple = Cache(), Cache()
    n = 0
    for i, x in enumerate(march_points(ps, target, prm.march_step)):
        n += 1
        s, m = interpolate(single, x), interpolate(multiple, x)
        if s is None or m is None:
            _, (rs, rm) = compute_pair(ps, x, prm, seed_seq(prm.seed, 401, i), adjacency_fn)
            if s is None:
                single.records.append(rs)
            if m is None:
                multiple.records.append(rm)
    return single, multiple, n


def render_field(ps, target: dict, single: Cache, multiple: Cache, prm: RenderParams, frozen=True):
    """FieldGrid render (src/renderer.py:425-437 with _point_value :335-368) → (image, stats)."""
    nx, ny = target["nx"], target["ny"]
    img = np.zeros((ny, nx, 3))
    stats = {"cache_hits": 0, "direct_evaluations": 0}
    pts = list(march_points(ps, target, prm.march_step))
    for j, x in enumerate(pts):
        iy, ix = divmod(j, nx)
        s, m = interpolate(single, x), interpolate(multiple, x)
        if s is not None and m is not None:
            stats["cache_hits"] += 1
            val = s + m
        else:
            stats["direct_evaluations"] += 1
            val, (rs, rm) = compute_pair(ps, x, prm, seed_seq(prm.seed, 307, iy, ix))
            if not frozen:
                if s is None:
                    single.records.append(rs)
                if m is None:
                    multiple.records.append(rm)
                a, b = interpolate(single, x), interpolate(multiple, x)
                if a is not None and b is not None:
                    val = a + b
        img[iy, ix] = 2.0 * np.pi * val
    return img, stats
