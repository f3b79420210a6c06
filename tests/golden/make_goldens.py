"""Generate golden fixtures by running the REFERENCE implementation (build container only).

Usage (from the repo root, in the container that mounts /root/reference):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_goldens.py

The reference package is imported read-only from /root/reference/pkg/src; nothing
is written there.  Outputs go to tests/golden/*.npz together with the numpy /
scipy versions that produced them (numpy PCG64/SeedSequence and scipy qhull are
the reference's unpinned third-party dependencies).  The GPU box
never runs this script; it only reads the committed .npz files.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import scipy

REF = Path("/root/reference/pkg/src")
REPO = Path(__file__).resolve().parents[2]
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))
sys.path.insert(0, str(REPO))

import volcache.renderer as vr  # noqa: E402
import volcache.subdivision as vs  # noqa: E402
from volcache import cache as vcache  # noqa: E402
from volcache import formfactor as vff  # noqa: E402
from volcache import scene as vscene  # noqa: E402

from paper_1805_09258_b200 import configs  # noqa: E402
from paper_1805_09258_b200.scene import scene_arrays, scene_to_dict  # noqa: E402

VERSIONS = np.array([np.__version__, scipy.__version__])


def ref_scene(scene):
    d = scene_to_dict(scene)
    d.pop("lights", None)  # extension key the reference does not know
    return vscene.scene_from_dict(d)


def scene_fields(prefix, scene):
    dim, V, E, A = scene_arrays(scene)
    return {
        f"{prefix}verts": V,
        f"{prefix}emission": E,
        f"{prefix}albedo": A,
        f"{prefix}bmin": np.asarray(scene.bounds_min, float),
        f"{prefix}bmax": np.asarray(scene.bounds_max, float),
        f"{prefix}sigma": np.array([scene.medium.sigma_s, scene.medium.sigma_a]),
    }


# ---------------------------------------------------------------------------


def gen_formfactors():
    rng = np.random.default_rng(1234)
    m = 256
    x2 = rng.uniform(-1, 1, (m, 2))
    y0 = rng.uniform(-1, 1, (m, 2))
    y1 = rng.uniform(-1, 1, (m, 2))
    y1[:8] = y0[:8] + 1e-7 * rng.normal(size=(8, 2))  # thin → degenerate γ
    y0[8:12] = x2[8:12]  # vertex coincidence
    ok2, v2, g2, h2 = vff.ff_segment_derivs_batch(x2, y0, y1)
    x3 = rng.uniform(-1, 1, (m, 3))
    t1 = rng.uniform(-1, 1, (m, 3))
    t2 = rng.uniform(-1, 1, (m, 3))
    t3 = rng.uniform(-1, 1, (m, 3))
    t3[:8] = x3[:8] + 0.3 * (t1[:8] - x3[:8]) + 0.6 * (t2[:8] - x3[:8])  # coplanar with x
    t1[8:12] = x3[8:12]
    ok3, v3, g3, h3 = vff.ff_triangle_derivs_batch(x3, t1, t2, t3)
    np.savez_compressed(
        OUT / "formfactors.npz", versions=VERSIONS,
        seg_x=x2, seg_y0=y0, seg_y1=y1, seg_ok=ok2, seg_val=v2, seg_grad=g2, seg_hess=h2,
        tri_x=x3, tri_y1=t1, tri_y2=t2, tri_y3=t3, tri_ok=ok3, tri_val=v3, tri_grad=g3, tri_hess=h3,
    )


def gen_trace():
    out = {"versions": VERSIONS}
    rng = np.random.default_rng(99)
    cases = {
        "c1": configs.cfg1_scene(),
        "c2": configs.cfg2_scene(),
        "room": configs.cfg3_scene(n_spheres=4, level=1),
    }
    for name, sc in cases.items():
        rs = ref_scene(sc)
        d = rs.dim
        m = 2048
        o = rng.uniform(rs.bounds_min, rs.bounds_max, (m, d))
        dirs = rng.normal(size=(m, d))
        dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
        s, idx = vscene.trace_or_bounds(rs, o, dirs)
        out.update(scene_fields(f"{name}_", sc))
        out[f"{name}_o"] = o
        out[f"{name}_d"] = dirs
        out[f"{name}_s"] = s
        out[f"{name}_idx"] = idx
    np.savez_compressed(OUT / "trace.npz", **out)


class Capture:
    """Monkeypatch hooks recording the direction set and primary trace of one build."""

    def __init__(self, inject=None):
        self.inject = inject
        self.dirs = None
        self.s = None
        self.idx = None

    def __enter__(self):
        self._sd = vs.stratified_directions
        self._tb = vs.trace_or_bounds
        cap = self

        def sd(dim, n, rng_seed=None, jitter=True):
            ds = cap._sd(dim, n, rng_seed, jitter)
            if cap.inject is not None:
                ds = vscene.DirectionSet(ds.dim, ds.directions, np.asarray(cap.inject), ds.stratum_measure)
            cap.dirs = ds
            return ds

        def tb(scene, o, d):
            s, idx = cap._tb(scene, o, d)
            if cap.s is None:
                cap.s, cap.idx = s, idx
            return s, idx

        vs.stratified_directions = sd
        vs.trace_or_bounds = tb
        return self

    def __exit__(self, *a):
        vs.stratified_directions = self._sd
        vs.trace_or_bounds = self._tb


def canonical_rotation(adj):
    """Rotate each simplex so its smallest index comes first (keeps orientation)."""
    adj = np.asarray(adj)
    k = np.argmin(adj, axis=1)
    return np.stack([adj[np.arange(len(adj)), (k + j) % 3] for j in range(3)], axis=1)


def gen_records(only=None):
    bundled = Path("/root/reference/pkg/scenes")
    pen = vscene.load_scene(bundled / "penumbra2d.json")
    box = vscene.load_scene(bundled / "box3d.json")
    c1 = configs.cfg1()
    c2 = configs.cfg2()
    refl2d = configs.cfg1_scene()
    refl2d = type(refl2d)(
        tuple(
            type(s)(vertices=s.vertices, emission=s.emission, albedo=(0.0 if s.is_emitter else 0.6))
            for s in refl2d.surfaces
        ),
        refl2d.medium, refl2d.bounds_min, refl2d.bounds_max,
    )
    box_refl = vscene.Scene(
        surfaces=tuple(
            vscene.Surface(vertices=s.vertices, emission=s.emission, albedo=(0.0 if s.is_emitter else 0.5))
            for s in box.surfaces
        ),
        medium=box.medium, bounds_min=box.bounds_min, bounds_max=box.bounds_max,
    )
    room = configs.cfg3_scene(n_spheres=4, level=1)
    room_pts = np.random.default_rng(2).uniform(room.bounds_min, room.bounds_max, (2, 3))
    # name: (scene, points, cfg_seed, n_angular, march_step, n_inner, n_light, inject_canonical)
    cases = {
        "cfg1_surf": (c1.scene, c1.points[:8], 0, 1024, 4.0, 1, 16, False),
        "cfg1_m01": (c1.scene, c1.points[:4], 0, 1024, 0.1, 1, 16, False),
        "pen2d": (pen, np.array([[0.15, 0.6], [0.5, 0.35], [0.3, 0.45], [0.8, 0.2]]), 7, 256, 0.05, 2, 16, False),
        "refl2d": (refl2d, c1.points[:4], 0, 256, 0.1, 1, 16, False),
        "cfg2_surf": (c2.scene, c2.points[:4], 1, 4096, 4.0, 1, 16, False),
        "cfg2_m01": (c2.scene, c2.points[:3], 1, 4096, 0.1, 1, 16, False),
        "cfg2_m01_canon": (c2.scene, c2.points[:3], 1, 4096, 0.1, 1, 16, True),
        "box3d_refl": (box_refl, np.array([[0.5, 0.5, 0.5], [0.2, 0.7, 0.3]]), 5, 256, 0.25, 2, 4, False),
        "room_small": (room, room_pts, 2, 1024, 0.2, 1, 16, False),
        # reflective walls: surface and media-gather hits lit by shadow rays (a3)
        "room_refl": (configs.cfg3_scene(n_spheres=4, level=1, wall_albedo=0.5), room_pts, 2, 1024, 0.2, 1, 4,
                      False),
    }
    for name, (sc, pts, cseed, n, step, n_inner, n_light, canon) in cases.items():
        if only and name not in only:
            continue
        rs = sc if isinstance(sc, vscene.Scene) else ref_scene(sc)
        N, d = pts.shape
        res = {k: [] for k in ("L", "grad", "hess", "stats", "dirs", "adj", "s", "idx",
                               "rec_value", "rec_grad", "rec_axes", "rec_radii", "rec_iso_radii")}
        for i in range(N):
            seed = vr._seed(cseed, 401, i)
            inject = None
            if canon:
                with Capture() as c0:
                    vs.build_subdivision(rs, pts[i], n_angular=n, march_step=step,
                                         rng_seed=vr._seed(cseed, 401, i), n_inner=n_inner,
                                         n_light_samples=n_light)
                inject = canonical_rotation(c0.dirs.adjacency)
            with Capture(inject) as cap:
                sub = vs.build_subdivision(rs, pts[i], n_angular=n, march_step=step, rng_seed=seed,
                                           n_inner=n_inner, n_light_samples=n_light)
            single, multiple, stats = vs.assemble_moments(sub, rs.medium)
            res["L"].append([single.L, multiple.L])
            res["grad"].append([single.grad, multiple.grad])
            res["hess"].append([single.hess, multiple.hess])
            res["stats"].append([stats["elements_evaluated"], stats["elements_dropped"], stats["star_vertices"]])
            res["dirs"].append(cap.dirs.directions)
            res["adj"].append(cap.dirs.adjacency)
            res["s"].append(cap.s)
            res["idx"].append(cap.idx)
            rv, rg, ra, rr, ri = [], [], [], [], []
            for mom in (single, multiple):
                rec = vcache.make_record(pts[i], mom, 0.05, rs.scale, rs.max_emission, anisotropic=True)
                iso = vcache.make_record(pts[i], mom, 0.05, rs.scale, rs.max_emission, anisotropic=False)
                rv.append(rec.value)
                rg.append(rec.grad)
                ra.append(rec.axes)
                rr.append(rec.radii)
                ri.append(iso.radii)
            res["rec_value"].append(rv)
            res["rec_grad"].append(rg)
            res["rec_axes"].append(ra)
            res["rec_radii"].append(rr)
            res["rec_iso_radii"].append(ri)
        out = {k: np.array(v) for k, v in res.items()}
        out.update(scene_fields("", rs))
        out.update(
            versions=VERSIONS, points=pts, cfg_seed=np.array(cseed),
            params=np.array([n, step, n_inner, n_light, 1.0 if canon else 0.0]),
        )
        np.savez_compressed(OUT / f"rec_{name}.npz", **out)
        print("wrote", name, flush=True)


def gen_make_record():
    """Eigen/radii edge cases through the reference make_record."""
    rng = np.random.default_rng(77)
    cases = []
    for dim in (2, 3):
        for kind in ("random", "zero", "rank1", "repeated", "negdef", "tiny", "diag"):
            for _ in range(4):
                L = rng.uniform(0.0, 3.0, 3)
                g = rng.normal(size=(3, dim))
                if kind == "random":
                    H = rng.normal(size=(3, dim, dim))
                elif kind == "zero":
                    H = np.zeros((3, dim, dim))
                elif kind == "rank1":
                    v = rng.normal(size=dim)
                    H = np.einsum("c,i,j->cij", rng.uniform(0.5, 2, 3), v, v)
                elif kind == "repeated":
                    H = np.broadcast_to(np.eye(dim) * rng.uniform(-2, 2), (3, dim, dim)).copy()
                    H[:, 0, 0] += 1e-9
                elif kind == "negdef":
                    Q = np.linalg.qr(rng.normal(size=(dim, dim)))[0]
                    H = np.broadcast_to(-Q @ np.diag(rng.uniform(1, 5, dim)) @ Q.T, (3, dim, dim)).copy()
                elif kind == "tiny":
                    H = 1e-20 * rng.normal(size=(3, dim, dim))
                else:
                    H = np.broadcast_to(np.diag(rng.uniform(-3, 3, dim)), (3, dim, dim)).copy()
                H = 0.5 * (H + np.swapaxes(H, 1, 2))
                if kind == "zero" and rng.random() < 0.5:
                    L = np.zeros(3)
                cases.append((dim, L, g, H))
    out = {"versions": VERSIONS}
    for j, (dim, L, g, H) in enumerate(cases):
        x = rng.uniform(0, 1, dim)
        mom = vs.Moments(L=L, grad=g, hess=H, kind="single")
        scale = float(np.sqrt(dim))
        for aniso in (True, False):
            for max_em in (10.0, 0.0):
                rec = vcache.make_record(x, mom, 0.05, scale, max_em, anisotropic=aniso)
                key = f"c{j}_{int(aniso)}_{int(max_em)}"
                out[key + "_axes"] = rec.axes
                out[key + "_radii"] = rec.radii
        out[f"c{j}_dim"] = np.array(dim)
        out[f"c{j}_x"] = x
        out[f"c{j}_L"] = L
        out[f"c{j}_g"] = g
        out[f"c{j}_H"] = H
    out["n_cases"] = np.array(len(cases))
    np.savez_compressed(OUT / "make_record.npz", **out)


def _rotation(dim, rng):
    q, r = np.linalg.qr(rng.normal(size=(dim, dim)))
    return q * np.sign(np.diag(r))[None, :]


def gen_interpolate():
    out = {"versions": VERSIONS}
    for dim in (2, 3):
        rng = np.random.default_rng(500 + dim)
        cache = vcache.RadianceCache(np.zeros(dim), np.ones(dim))
        recs = []
        for _ in range(40):
            rec = vcache.CacheRecord(
                position=rng.uniform(0, 1, dim), value=rng.uniform(0, 5, 3),
                grad=rng.normal(size=(3, dim)), axes=_rotation(dim, rng),
                radii=rng.uniform(0.02, 0.25 * np.sqrt(dim), dim),
            )
            cache.insert(rec)
            recs.append(rec)
        # power-of-two record for the exclusive-boundary case (tests/test_cache.py:586-594)
        edge = vcache.CacheRecord(position=np.full(dim, 0.5), value=np.ones(3), grad=np.zeros((3, dim)),
                                  axes=np.eye(dim), radii=np.full(dim, 0.125))
        cache.insert(edge)
        recs.append(edge)
        q = rng.uniform(-0.2, 1.2, (400, dim))
        q[0] = 0.5
        q[1] = 0.5
        q[1, 0] = 0.625
        J = np.full((len(q), 3), np.nan)
        cnt = np.zeros(len(q), np.int64)
        for i, x in enumerate(q):
            v = vcache.interpolate(cache, x)
            cnt[i] = len(cache.query(x))
            if v is not None:
                J[i] = v
        out[f"d{dim}_pos"] = np.array([r.position for r in recs])
        out[f"d{dim}_value"] = np.array([r.value for r in recs])
        out[f"d{dim}_grad"] = np.array([r.grad for r in recs])
        out[f"d{dim}_axes"] = np.array([r.axes for r in recs])
        out[f"d{dim}_radii"] = np.array([r.radii for r in recs])
        out[f"d{dim}_q"] = q
        out[f"d{dim}_J"] = J
        out[f"d{dim}_count"] = cnt
    np.savez_compressed(OUT / "interpolate.npz", **out)


def gen_render():
    """Tiny frozen-cache camera render of the small window room (src/renderer.py:402-484)."""
    sc = configs.cfg3_scene(n_spheres=4, level=1)
    rs = ref_scene(sc)
    cam = vr.Camera(position=np.array([2.0, 1.5, 0.2]), look_at=np.array([2.0, 1.5, 4.0]),
                    up=np.array([0.0, 1.0, 0.0]), fov_degrees=60.0, width=8, height=5)
    st = vr.RenderSettings(mode="ours-aniso", epsilon=0.5, spp=1, march_step=0.5, n_angular=256,
                           seed=3, frozen=True, n_inner=1, n_light_samples=16)
    cs, pop = vr.populate_cache(rs, cam, st)
    img, stats = vr.render(rs, cam, st, cache_set=cs)
    out = {"versions": VERSIONS, "image": img}
    out.update(scene_fields("", sc))
    for kind, c in (("single", cs.single), ("multiple", cs.multiple)):
        recs = c.records
        out[f"{kind}_pos"] = np.array([r.position for r in recs])
        out[f"{kind}_value"] = np.array([r.value for r in recs])
        out[f"{kind}_grad"] = np.array([r.grad for r in recs])
        out[f"{kind}_axes"] = np.array([r.axes for r in recs])
        out[f"{kind}_radii"] = np.array([r.radii for r in recs])
    out["stats"] = np.array([stats["cache_hits"], stats["direct_evaluations"], pop["points_marched"]])
    out["settings"] = np.array([st.epsilon, st.spp, st.march_step, st.n_angular, st.seed, st.n_inner,
                                st.n_light_samples])
    out["camera"] = np.concatenate([cam.position, cam.look_at, cam.up,
                                    [cam.fov_degrees, cam.width, cam.height]])
    np.savez_compressed(OUT / "render.npz", **out)


def _records_fields(prefix, cache):
    recs = cache.records
    d = cache.bounds_min.size
    def row(r):
        if hasattr(r, "radius"):  # BaselineRecord sphere → identity axes, equal radii (device layout)
            return np.concatenate([r.position, r.value, r.grad.ravel(), np.eye(d).ravel(), np.full(d, r.radius)])
        return np.concatenate([r.position, r.value, r.grad.ravel(), r.axes.ravel(), r.radii])

    rows = [row(r) for r in recs]
    return {prefix: np.array(rows).reshape(len(rows), d + 3 + 3 * d + d * d + d)}


def gen_populate():
    """populate_cache / field render / camera render through the reference (src/renderer.py:282-484)."""
    bundled = Path("/root/reference/pkg/scenes")
    pen = vscene.load_scene(bundled / "penumbra2d.json")
    box = vscene.load_scene(bundled / "box3d.json")
    simple = vscene.Scene(
        surfaces=(vscene.Surface(vertices=np.array([[0.2, 0.8], [0.8, 0.8]]), emission=np.array([5.0, 4.0, 3.0])),),
        medium=vscene.Medium(sigma_s=0.5, sigma_a=0.25), bounds_min=np.zeros(2), bounds_max=np.ones(2))
    cheap = dict(mode="ours-aniso", epsilon=0.05, march_step=0.1, n_angular=64, n_light_samples=4, seed=3)
    cam3d = dict(mode="ours-aniso", epsilon=0.2, march_step=0.25, n_angular=512, n_light_samples=4, spp=1, seed=5)
    out = {"versions": VERSIONS}
    out.update(scene_fields("simple_", simple))
    out.update(scene_fields("pen_", pen))
    out.update(scene_fields("box_", box))

    def settings_vec(st):
        return np.array([st.epsilon, st.march_step, st.n_angular, st.n_light_samples, st.seed, st.n_inner, st.spp,
                         1.0 if st.frozen else 0.0, 1.0 if st.mode == "ours-iso" else 0.0])

    def pop(name, scene, target, st):
        cs, stats = vr.populate_cache(scene, target, st)
        out.update(_records_fields(f"{name}_single", cs.single))
        out.update(_records_fields(f"{name}_multiple", cs.multiple))
        out[f"{name}_stats"] = np.array([stats["points_marched"], stats["records_single"], stats["records_multiple"]])
        out[f"{name}_settings"] = settings_vec(st)
        print("populate", name, stats, flush=True)
        return cs

    def field(nx, ny, scene):
        return vr.FieldGrid.for_scene(scene, nx, ny)

    # populate: FieldGrid targets
    pop("simple6", simple, field(6, 6, simple), vr.RenderSettings(**cheap))
    pop("pen8_tight", pen, field(8, 8, pen), vr.RenderSettings(**{**cheap, "epsilon": 0.005}))
    pop("pen8_loose", pen, field(8, 8, pen), vr.RenderSettings(**{**cheap, "epsilon": 0.5}))
    pop("pen16_iso", pen, field(16, 12, pen), vr.RenderSettings(**{**cheap, "mode": "ours-iso", "seed": 8}))
    # field renders: default (populate then frozen lookups), frozen with an empty cache, growing cache
    st = vr.RenderSettings(**{**cheap, "seed": 11})
    img, stats = vr.render(pen, field(6, 5, pen), st)
    out["render_pen65_image"] = img
    out["render_pen65_stats"] = np.array([stats["cache_hits"], stats["direct_evaluations"], stats["records"]])
    out["render_pen65_settings"] = settings_vec(st)
    st = vr.RenderSettings(**{**cheap, "frozen": True})
    empty = vr.CacheSet(simple, "ours-aniso")
    img, stats = vr.render(simple, field(3, 3, simple), st, cache_set=empty)
    out["render_frozen_image"] = img
    out["render_frozen_stats"] = np.array([stats["cache_hits"], stats["direct_evaluations"], empty.record_count])
    out["render_frozen_settings"] = settings_vec(st)
    st = vr.RenderSettings(**{**cheap, "frozen": False})
    growing = vr.CacheSet(simple, "ours-aniso")
    img, stats = vr.render(simple, field(6, 6, simple), st, cache_set=growing)
    out["render_grow_image"] = img
    out["render_grow_stats"] = np.array([stats["cache_hits"], stats["direct_evaluations"], growing.record_count])
    out["render_grow_settings"] = settings_vec(st)
    out.update(_records_fields("render_grow_single", growing.single))
    out.update(_records_fields("render_grow_multiple", growing.multiple))
    # camera targets over box3d
    cam = vr.Camera(position=np.array([0.5, 0.5, 0.5]), look_at=np.array([0.5, 0.5, 1.0]),
                    up=np.array([0.0, 1.0, 0.0]), fov_degrees=60.0, width=3, height=2)
    st = vr.RenderSettings(**cam3d)
    cs = pop("box32", box, cam, st)
    img, stats = vr.render(box, cam, st, cache_set=cs)
    out["box32_image"] = img
    out["box32_camera"] = np.concatenate([cam.position, cam.look_at, cam.up, [cam.fov_degrees, cam.width,
                                                                                cam.height]])
    cam = vr.Camera(position=np.array([0.5, 0.3, 0.05]), look_at=np.array([0.5, 0.5, 1.0]),
                    up=np.array([0.0, 1.0, 0.0]), fov_degrees=70.0, width=10, height=8)
    st = vr.RenderSettings(**{**cam3d, "march_step": 0.1, "n_angular": 128, "epsilon": 0.1, "seed": 9})
    pop("box108", box, cam, st)
    out["box108_camera"] = np.concatenate([cam.position, cam.look_at, cam.up, [cam.fov_degrees, cam.width,
                                                                                 cam.height]])
    # larger targets: many speculative windows on the device
    pop("pen64", pen, field(64, 48, pen), vr.RenderSettings(**{**cheap, "epsilon": 0.01, "seed": 21}))
    cam = vr.Camera(position=np.array([0.1, 0.2, 0.05]), look_at=np.array([0.6, 0.5, 1.0]),
                    up=np.array([0.0, 1.0, 0.0]), fov_degrees=75.0, width=32, height=24)
    st = vr.RenderSettings(**{**cam3d, "march_step": 0.05, "n_angular": 256, "epsilon": 0.05, "seed": 13})
    pop("box3224", box, cam, st)
    out["box3224_camera"] = np.concatenate([cam.position, cam.look_at, cam.up, [cam.fov_degrees, cam.width,
                                                                                  cam.height]])
    np.savez_compressed(OUT / "populate.npz", **out)


def gen_io():
    """A cache document and a PFM written by the reference's own writers (src/cache.py:441-457,
    src/renderer.py:689-699)."""
    cache = vcache.RadianceCache(np.array([0.0, -1.0]), np.array([2.0, 3.0]))
    c, s_ = np.cos(0.4), np.sin(0.4)
    cache.insert(vcache.CacheRecord(position=np.array([0.5, 0.5]), value=np.array([1.0, 0.5, 0.25]),
                                    grad=np.arange(6.0).reshape(3, 2) / 7.0, axes=np.array([[c, -s_], [s_, c]]),
                                    radii=np.array([0.2, 0.1])))
    cache.insert(vcache.BaselineRecord(position=np.array([1.0, 2.0]), value=np.array([0.5, 0.25, 0.125]),
                                       grad=np.ones((3, 2)), radius=0.15))
    vcache.save_cache(cache, OUT / "ref_cache.json", metadata={"mode": "test", "epsilon": 0.01})
    img = np.random.default_rng(0).uniform(0.0, 10.0, size=(5, 7, 3)).astype(np.float32)
    vr.write_pfm(OUT / "ref_image.pfm", img)


def gen_baseline():
    """baseline_estimate / make_baseline_record / log_space_interpolate and the baseline
    cache mode through the reference (src/subdivision.py:416-521, src/cache.py:190-394)."""
    bundled = Path("/root/reference/pkg/scenes")
    pen = vscene.load_scene(bundled / "penumbra2d.json")
    box = vscene.load_scene(bundled / "box3d.json")
    box_refl = vscene.Scene(
        surfaces=tuple(vscene.Surface(vertices=s.vertices, emission=s.emission,
                                      albedo=(0.0 if s.is_emitter else 0.5)) for s in box.surfaces),
        medium=box.medium, bounds_min=box.bounds_min, bounds_max=box.bounds_max)
    out = {"versions": VERSIONS}
    out.update(scene_fields("pen_", pen))
    out.update(scene_fields("box_", box))
    out.update(scene_fields("boxr_", box_refl))
    cases = {  # name: (scene prefix, scene, points, n_angular, max_media_bounces, n_light)
        "pen": ("pen_", pen, np.array([[0.15, 0.6], [0.3, 0.45], [0.8, 0.2]]), 512, 2, 16),
        "pen3": ("pen_", pen, np.array([[0.5, 0.35]]), 256, 4, 8),
        "box": ("box_", box, np.array([[0.5, 0.5, 0.5], [0.2, 0.7, 0.3]]), 1024, 2, 8),
        "boxr": ("boxr_", box_refl, np.array([[0.4, 0.6, 0.5]]), 512, 3, 4),
    }
    for name, (prefix, sc, pts, n, mmb, nl) in cases.items():
        vals, grads, svals, snorms, radii = [], [], [], [], []
        for i, x in enumerate(pts):
            s_, m_ = vs.baseline_estimate(sc, x, n_angular=n, rng_seed=vr._seed(17, 401, i), max_media_bounces=mmb,
                                          n_light_samples=nl)
            vals.append([s_.value, m_.value])
            grads.append([s_.grad, m_.grad])
            svals.append([s_.sample_values, m_.sample_values])
            snorms.append([s_.sample_grad_norms, m_.sample_grad_norms])
            radii.append([vcache.make_baseline_record(x, e, sc.scale, 0.7).radius for e in (s_, m_)])
        out[f"{name}_points"] = pts
        out[f"{name}_params"] = np.array([n, mmb, nl])
        out[f"{name}_value"] = np.array(vals)
        out[f"{name}_grad"] = np.array(grads)
        out[f"{name}_svals"] = np.array(svals)
        out[f"{name}_snorms"] = np.array(snorms)
        out[f"{name}_radius"] = np.array(radii)
        out[f"{name}_prefix"] = np.array(prefix)
    # log-space interpolation on a random sphere-record cache
    rng = np.random.default_rng(808)
    cache = vcache.RadianceCache(np.zeros(3), np.ones(3))
    recs = []
    for _ in range(40):
        v = rng.uniform(0.0, 2.0, 3)
        v[rng.uniform(size=3) < 0.2] = 0.0
        r = vcache.BaselineRecord(position=rng.uniform(0, 1, 3), value=v, grad=rng.normal(size=(3, 3)),
                                  radius=float(rng.uniform(0.05, 0.3)))
        cache.insert(r)
        recs.append(np.concatenate([r.position, r.value, r.grad.ravel(), [r.radius]]))
    q = rng.uniform(0, 1, (300, 3))
    J = np.array([vcache.log_space_interpolate(cache, x) if vcache.log_space_interpolate(cache, x) is not None
                  else np.full(3, np.nan) for x in q])
    out["log_records"] = np.array(recs)
    out["log_q"] = q
    out["log_J"] = J
    # baseline cache mode: populate + field render (2D), camera populate (3D)
    cheap = dict(mode="baseline", epsilon=0.05, march_step=0.1, n_angular=64, n_light_samples=4, seed=3,
                 baseline_alpha=0.8)
    st = vr.RenderSettings(**cheap)
    grid = vr.FieldGrid.for_scene(pen, 8, 6)
    cs, pst = vr.populate_cache(pen, grid, st)
    out.update(_records_fields("bpop_single", cs.single))
    out.update(_records_fields("bpop_multiple", cs.multiple))
    img, rst = vr.render(pen, grid, st, cache_set=cs)
    out["bpop_image"] = img
    out["bpop_stats"] = np.array([pst["points_marched"], pst["records_single"], pst["records_multiple"],
                                  rst["cache_hits"], rst["direct_evaluations"]])
    cam = vr.Camera(position=np.array([0.5, 0.3, 0.05]), look_at=np.array([0.5, 0.5, 1.0]),
                    up=np.array([0.0, 1.0, 0.0]), fov_degrees=70.0, width=6, height=5)
    st3 = vr.RenderSettings(mode="baseline", epsilon=0.1, march_step=0.1, n_angular=256, n_light_samples=4, seed=9,
                            spp=1)
    cs3, pst3 = vr.populate_cache(box, cam, st3)
    out.update(_records_fields("bcam_single", cs3.single))
    out.update(_records_fields("bcam_multiple", cs3.multiple))
    img3, rst3 = vr.render(box, cam, st3, cache_set=cs3)
    out["bcam_image"] = img3
    out["bcam_stats"] = np.array([pst3["points_marched"], pst3["records_single"], pst3["records_multiple"],
                                  rst3["cache_hits"], rst3["direct_evaluations"]])
    out["bcam_camera"] = np.concatenate([cam.position, cam.look_at, cam.up, [cam.fov_degrees, cam.width,
                                                                               cam.height]])
    np.savez_compressed(OUT / "baseline.npz", **out)


def gen_baseline_rng():
    """baseline_estimate called twice on ONE Generator (src/subdivision.py:431): the second
    call sees the stream the first left behind, and the draw after both pins how many
    doubles the reference consumed (its collision loop stops at the first bounce without a
    collision, src/subdivision.py:480-486)."""
    bundled = Path("/root/reference/pkg/scenes")
    pen = vscene.load_scene(bundled / "penumbra2d.json")
    box = vscene.load_scene(bundled / "box3d.json")
    out = {"versions": VERSIONS}
    out.update(scene_fields("pen_", pen))
    out.update(scene_fields("box_", box))
    cases = {  # name: (prefix, scene, points, n, max_media_bounces, generator seed)
        "pen": ("pen_", pen, np.array([[0.15, 0.6], [0.3, 0.45]]), 256, 2, 71),
        "pen6": ("pen_", pen, np.array([[0.5, 0.35], [0.7, 0.7]]), 64, 6, 72),
        "box": ("box_", box, np.array([[0.5, 0.5, 0.5], [0.2, 0.7, 0.3]]), 512, 3, 73),
        "box9": ("box_", box, np.array([[0.4, 0.3, 0.6]]), 16, 9, 74),
    }
    for name, (prefix, sc, pts, n, mmb, gs) in cases.items():
        g = np.random.default_rng(gs)
        vals = []
        for x in pts:
            s_, m_ = vs.baseline_estimate(sc, x, n_angular=n, rng_seed=g, max_media_bounces=mmb, n_light_samples=4)
            vals.append([np.concatenate([s_.value, s_.grad.ravel()]), np.concatenate([m_.value, m_.grad.ravel()])])
        out[f"{name}_prefix"] = np.array(prefix)
        out[f"{name}_points"] = pts
        out[f"{name}_params"] = np.array([n, mmb, gs])
        out[f"{name}_est"] = np.array(vals)
        out[f"{name}_next"] = np.array(g.random())
    np.savez_compressed(OUT / "baseline_rng.npz", **out)


def _chunked_trace(orig, chunk=64):
    """Per-ray identical stand-in for scene.trace that bounds numpy's (m, K, 3) temporaries
    (SURVEY.md §8d chunked-trace shim): the reference's own function on ray chunks."""
    def trace(scene, origins, dirs, t_max=None):
        origins, dirs = np.asarray(origins, float), np.asarray(dirs, float)
        m = origins.shape[0]
        s = np.empty(m)
        idx = np.empty(m, dtype=np.int64)
        for a in range(0, m, chunk):
            tm = None if t_max is None else (t_max if np.ndim(t_max) == 0 else np.asarray(t_max)[a:a + chunk])
            s[a:a + chunk], idx[a:a + chunk] = orig(scene, origins[a:a + chunk], dirs[a:a + chunk], tm)
        return s, idx
    return trace


def _hg_sample_ref(g, cur, u0, u1):
    """HG direction sampling about `cur` (the extension's convention)."""
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


def _gather_bounces_shim(seed_box, bounces, hg=0.0, inscatter=None):
    """Extension oracle written with the reference's own primitives: mean_surface_gather
    (src/transport.py:288-310) continued by up to `bounces` − 1 media scattering events per
    gather path, exactly the multiple-scattering loop of path_trace_radiance
    (src/transport.py:362-388); per path and bounce the draws (u_dist, u0, u1) come from the
    record's stream continued after every draw build_subdivision makes (2·n directions,
    then 2·n_inner per media sample)."""
    import volcache.transport as vt

    def gather(scene, points, dirs_per_point, n_light_samples=16):
        m, n, dim = dirs_per_point.shape
        per_dir = 2 if dim == 3 else 1  # draws per stratum jitter and per gather direction
        g = np.random.default_rng(seed_box["seed"])
        g.bit_generator.advance(per_dir * seed_box["n_dirs"] + per_dir * m * n)
        ex = g.random((m * n, bounces - 1, 3 if dim == 3 else 2))
        origins = np.repeat(points, n, axis=0)
        dirs = dirs_per_point.reshape(-1, dim)
        s, idx = vscene.trace_or_bounds(scene, origins, dirs)
        tot = np.exp(-scene.medium.sigma_t * s)[:, None] * vt.surface_radiance_batch(
            scene, idx, origins + s[:, None] * dirs, dirs, n_light_samples)
        sig_t, sig_s = scene.medium.sigma_t, scene.medium.sigma_s
        w0 = np.ones(m * n)
        if hg != 0.0:  # HG scattering at the media sample toward the cache point
            dx = origins - seed_box["x"][None]
            wk = dx / np.sqrt((dx * dx).sum(axis=1))[:, None]
            c = (dirs * wk).sum(axis=1)
            w0 = 4.0 * np.pi * ((1.0 - hg * hg) / (4.0 * np.pi * (1.0 + hg * hg - 2.0 * hg * c) ** 1.5))
            tot = tot * w0[:, None]
        w = w0.copy()
        alive = np.ones(m * n, dtype=bool)
        pos, cur_d, cur_s = origins, dirs, s
        for b in range(bounces - 1):
            t = -np.log1p(-ex[:, b, 0]) / sig_t
            collide = alive & (t < cur_s)
            if not np.any(collide):
                break
            pos = pos + np.where(collide, t, 0.0)[:, None] * cur_d
            w = w * np.where(collide, sig_s / sig_t, 1.0)
            if hg != 0.0:
                nd = _hg_sample_ref(hg, cur_d, ex[:, b, 1], ex[:, b, 2])
            else:
                nd = vt.uniform_directions(dim, ex[:, b, 1] if dim == 2 else ex[:, b, 1:3])
            s2 = np.zeros(m * n)
            s2[collide], idx2 = vscene.trace_or_bounds(scene, pos[collide], nd[collide])
            lo2 = vt.surface_radiance_batch(scene, idx2, pos[collide] + s2[collide, None] * nd[collide],
                                            nd[collide], n_light_samples)
            tot[collide] += w[collide, None] * np.exp(-sig_t * s2[collide])[:, None] * lo2
            if inscatter is not None:  # delta lights scattered at this collision toward −cur_d
                tot[collide] += w[collide, None] * inscatter(pos[collide], hg, cur_d[collide])
            alive = collide
            cur_d = nd
            cur_s = s2
        return tot.reshape(m, n, 3).mean(axis=1)

    return gather


def gen_media_hg():
    """Extension records with Henyey–Greenstein media (g = 0.5, BASELINE cfg3) and 4 media
    events per gather path: the reference's build_subdivision + assemble_moments with the
    gather rebuilt from its primitives (_gather_bounces_shim)."""
    room = configs.cfg3_scene(n_spheres=4, level=1)
    rs = ref_scene(room)
    pts = np.random.default_rng(23).uniform(room.bounds_min + 0.3, room.bounds_max - 0.3, (3, 3))
    n, step, B, g = 1024, 0.2, 4, 0.5
    box = {}
    orig = vs.mean_surface_gather
    vs.mean_surface_gather = _gather_bounces_shim(box, B, g)
    res = {k: [] for k in ("L", "grad", "hess", "stats", "adj")}
    try:
        for i, x in enumerate(pts):
            box.update(seed=vr._seed(4, 401, i), n_dirs=n, x=np.asarray(x, float))
            with Capture() as cap:
                sub = vs.build_subdivision(rs, x, n_angular=n, march_step=step, rng_seed=vr._seed(4, 401, i))
            single, multiple, stats = vs.assemble_moments(sub, rs.medium)
            res["L"].append([single.L, multiple.L])
            res["grad"].append([single.grad, multiple.grad])
            res["hess"].append([single.hess, multiple.hess])
            res["stats"].append([stats["elements_evaluated"], stats["elements_dropped"], stats["star_vertices"]])
            res["adj"].append(np.asarray(cap.dirs.adjacency, np.int32))
    finally:
        vs.mean_surface_gather = orig
    out = {k: np.array(v) for k, v in res.items()}
    out.update(scene_fields("", rs))
    out.update(versions=VERSIONS, points=pts, cfg_seed=np.array(4), params=np.array([n, step, 1, 16, float(B), g]))
    np.savez_compressed(OUT / "rec_media_hg.npz", **out)
    print("wrote media_hg", flush=True)


def gen_media_bounces():
    """Records with the ≤ B-bounce media-radiance extension (BASELINE cfg3 asks for up to 4;
    the reference has one extra bounce): the reference's build_subdivision + assemble_moments
    with mean_surface_gather replaced by _gather_bounces_shim (reference primitives only)."""
    room = configs.cfg3_scene(n_spheres=4, level=1)
    rs = ref_scene(room)
    pts = np.random.default_rng(21).uniform(room.bounds_min + 0.3, room.bounds_max - 0.3, (3, 3))
    n, step, B = 1024, 0.2, 4
    box = {}
    orig = vs.mean_surface_gather
    vs.mean_surface_gather = _gather_bounces_shim(box, B)
    res = {k: [] for k in ("L", "grad", "hess", "stats", "adj")}
    try:
        for i, x in enumerate(pts):
            box.update(seed=vr._seed(3, 401, i), n_dirs=n)
            with Capture() as cap:
                sub = vs.build_subdivision(rs, x, n_angular=n, march_step=step, rng_seed=vr._seed(3, 401, i))
            single, multiple, stats = vs.assemble_moments(sub, rs.medium)
            res["L"].append([single.L, multiple.L])
            res["grad"].append([single.grad, multiple.grad])
            res["hess"].append([single.hess, multiple.hess])
            res["stats"].append([stats["elements_evaluated"], stats["elements_dropped"], stats["star_vertices"]])
            res["adj"].append(np.asarray(cap.dirs.adjacency, np.int32))
    finally:
        vs.mean_surface_gather = orig
    out = {k: np.array(v) for k, v in res.items()}
    out.update(scene_fields("", rs))
    out.update(versions=VERSIONS, points=pts, cfg_seed=np.array(3), params=np.array([n, step, 1, 16, float(B)]))
    np.savez_compressed(OUT / "rec_media_bounces.npz", **out)
    print("wrote media_bounces", flush=True)


def _delta_ref(rs, lights):
    """Delta-light extension written with the reference's own primitives (scene.trace,
    scene.bounds_exit): per light the direction toward it, the attenuated geometric term with
    the reference's shadow-ray rule (src/transport.py:213-214), and its rgb strength."""
    dim = rs.dim
    off = 1e-6 * rs.scale
    sig = rs.medium.sigma_t

    def incident(org):
        org = np.atleast_2d(org)
        m = org.shape[0]
        res = []
        for row in lights:
            kind, v, I = int(row[0]), row[1:1 + dim], row[4:7]
            val = np.zeros(m)
            if kind == 0:
                to = v[None] - org
                r = np.linalg.norm(to, axis=1)
                ok = r > off
                d = np.zeros_like(to)
                d[ok] = to[ok] / r[ok, None]
                th, _ = vscene.trace(rs, org[ok], d[ok])
                vis = th >= r[ok] * (1.0 - 1e-6)
                ii = np.flatnonzero(ok)[vis]
                val[ii] = np.exp(-sig * r[ii]) / np.maximum(r[ii], off) ** (dim - 1)
            else:
                d = np.broadcast_to(v, (m, dim)).copy()
                th, _ = vscene.trace(rs, org, d)
                vis = ~np.isfinite(th)
                val[vis] = np.exp(-sig * vscene.bounds_exit(rs, org[vis], d[vis]))
            res.append((d, val, I))
        return res

    def inscatter(pts, g=0.0, toward=None):
        out = np.zeros((np.atleast_2d(pts).shape[0], 3))
        norm = 4.0 * np.pi if dim == 3 else 2.0 * np.pi
        for d, val, I in incident(pts):
            w = val / norm
            if g != 0.0:
                c = (d * toward).sum(axis=1)
                w = w * (4.0 * np.pi * ((1.0 - g * g) / (4.0 * np.pi * (1.0 + g * g - 2.0 * g * c) ** 1.5)))
            out += w[:, None] * I[None]
        return out

    def single(x):
        x = np.asarray(x, float)
        L, G, H = np.zeros(3), np.zeros((3, dim)), np.zeros((3, dim, dim))
        norm = 4.0 * np.pi if dim == 3 else 2.0 * np.pi
        c = rs.medium.sigma_s / norm / norm
        k = dim - 1
        for row, (d, val, I) in zip(lights, incident(x[None])):
            phi = val[0]
            if not phi > 0.0:
                continue
            if int(row[0]) == 0:
                w = x - row[1:1 + dim]
                r = float(np.linalg.norm(w))
                u = w / r
                a = sig + k / r
                d1, d2 = -a * phi, (a * a + k / (r * r)) * phi
                g = d1 * u
                h = d2 * np.outer(u, u) + d1 / r * (np.eye(dim) - np.outer(u, u))
            else:
                dv = d[0]
                with np.errstate(divide="ignore", invalid="ignore"):
                    t = np.maximum((rs.bounds_min - x) / dv, (rs.bounds_max - x) / dv)
                t = np.where(np.isnan(t), np.inf, t)
                ax = int(np.argmin(t))
                e = np.zeros(dim)
                e[ax] = 1.0 / dv[ax]
                g = sig * phi * e
                h = sig * sig * phi * np.outer(e, e)
            L += c * phi * I
            G += c * I[:, None] * g[None]
            H += c * I[:, None, None] * h[None]
        return L, G, H

    return incident, inscatter, single


def gen_delta_lights():
    """Extension records with delta lights (BASELINE.json cfg1/cfg2/cfg4 point lights, cfg3's
    directional light; the reference has area emitters only): the reference's build_subdivision
    + assemble_moments with direct_lighting and mean_surface_gather extended through the
    reference's own trace / bounds_exit (_delta_ref), plus the lights' closed-form single
    scattering at the cache point.  Four cases: 2D cfg1-as-specified with a reflective occluder;
    a reflective 3D room with open windows (directional + point); a non-reflective room with
    emissive portals and a point light (the two-pass gather); open windows with HG g = 0.5 and
    3 media events per gather path (delta lights scattered at every collision)."""
    import volcache.transport as vt
    from paper_1805_09258_b200.scene import directional_light, point_light

    sun = directional_light(configs.SUN_TOWARD, configs.SUN_IRRADIANCE)
    lamp = point_light((2.6, 2.2, 1.4), (6.0, 5.0, 4.0))
    cases = [
        ("d2", configs.cfg1_spec_scene(occluder_albedo=0.3), 4, 1024, 0.1, 1, 0.0, 41),
        ("refl", configs.cfg3_scene(4, 1, wall_albedo=0.5, open_windows=True, lights=[sun, lamp]), 3, 1024, 0.2, 1,
         0.0, 42),
        ("portal", configs.cfg3_scene(4, 1, lights=[lamp]), 2, 1024, 0.2, 1, 0.0, 43),
        ("hg", configs.cfg3_scene(4, 1, open_windows=True, lights=[sun, lamp]), 2, 1024, 0.2, 3, 0.5, 44),
    ]
    out = {"versions": VERSIONS}
    for name, sc, npts, n, step, B, g, seed in cases:
        rs = ref_scene(sc)
        dim = rs.dim
        incident, inscatter, single = _delta_ref(rs, sc.lights)
        pts = np.random.default_rng(seed).uniform(rs.bounds_min + 0.15 * (rs.bounds_max - rs.bounds_min),
                                                  rs.bounds_max - 0.15 * (rs.bounds_max - rs.bounds_min), (npts, dim))
        box = {}
        o_dl, o_msg = vt.direct_lighting, vs.mean_surface_gather

        def direct_lighting(scene, points, normals, n_light_samples=16, _o=o_dl, _inc=incident):
            points, normals = np.atleast_2d(points), np.atleast_2d(normals)
            base = _o(scene, points, normals, n_light_samples)
            add = np.zeros_like(base)
            for d, val, I in _inc(points + 1e-6 * scene.scale * normals):
                cp = np.clip(np.einsum("md,md->m", normals, d), 0.0, None)
                add += (cp * val)[:, None] * I[None]
            return base + add / (np.pi if scene.dim == 3 else 2.0)

        base_gather = o_msg if (B == 1 and g == 0.0) else _gather_bounces_shim(box, B, g, inscatter)

        def gather(scene, points, dirs_pp, n_light_samples=16, _b=base_gather, _ins=inscatter, _g=g):
            dx = points - box["x"][None]
            wk = dx / np.sqrt((dx * dx).sum(axis=1))[:, None]
            return _b(scene, points, dirs_pp, n_light_samples) + _ins(points, _g, wk)

        vt.direct_lighting = direct_lighting
        vs.mean_surface_gather = gather
        res = {k: [] for k in ("L", "grad", "hess", "stats", "adj")}
        try:
            for i, x in enumerate(pts):
                box.update(seed=vr._seed(seed, 401, i), n_dirs=n, x=np.asarray(x, float))
                with Capture() as cap:
                    sub = vs.build_subdivision(rs, x, n_angular=n, march_step=step, rng_seed=vr._seed(seed, 401, i))
                sg, mu, stats = vs.assemble_moments(sub, rs.medium)
                dL, dG, dH = single(x)
                res["L"].append([sg.L + dL, mu.L])
                res["grad"].append([sg.grad + dG, mu.grad])
                res["hess"].append([sg.hess + dH, mu.hess])
                res["stats"].append([stats["elements_evaluated"], stats["elements_dropped"], stats["star_vertices"]])
                res["adj"].append(np.asarray(cap.dirs.adjacency, np.int32))
        finally:
            vt.direct_lighting = o_dl
            vs.mean_surface_gather = o_msg
        out.update({f"{name}_{k}": np.array(v) for k, v in res.items()})
        out.update(scene_fields(f"{name}_", rs))
        out[f"{name}_lights"] = np.asarray(sc.lights, float)
        out[f"{name}_points"] = pts
        out[f"{name}_params"] = np.array([n, step, 1, 16, float(B), g, float(seed)])
        print("delta lights", name, np.array(res["L"])[:, :, 1].tolist(), flush=True)
    np.savez_compressed(OUT / "rec_delta_lights.npz", **out)


def gen_surface():
    """Per-hit outgoing radiance surface_radiance_batch (src/transport.py:240-254) on
    reflective rooms (walls albedo 0.5): the small room on 4096 random rays, the full cfg3
    room (51,300 triangles; chunked trace) on 48 rays; the hits from the reference's trace."""
    import volcache.transport as vt

    out = {"versions": VERSIONS}
    shim = _chunked_trace(vscene.trace, 16)
    saved = {m: m.trace for m in (vscene, vr, vt)}
    try:
        for mod in saved:
            mod.trace = shim
        for name, sc, m, seed in (("small", configs.cfg3_scene(n_spheres=4, level=1, wall_albedo=0.5), 4096, 31),
                                  ("full", configs.cfg3_scene(wall_albedo=0.5), 48, 32)):
            rs = ref_scene(sc)
            rng = np.random.default_rng(seed)
            o = rng.uniform(rs.bounds_min, rs.bounds_max, (m, 3))
            d = rng.normal(size=(m, 3))
            d /= np.linalg.norm(d, axis=1, keepdims=True)
            s_, idx = vscene.trace(rs, o, d)
            hit = o + np.where(np.isfinite(s_), s_, 0.0)[:, None] * d
            lo = vt.surface_radiance_batch(rs, idx, hit, d, 16)
            out[f"{name}_points"] = hit
            out[f"{name}_dirs"] = d
            out[f"{name}_idx"] = idx
            out[f"{name}_lo"] = lo
            print("surface", name, int((idx >= 0).sum()), "hits", flush=True)
    finally:
        for mod, f in saved.items():
            mod.trace = f
    np.savez_compressed(OUT / "surface.npz", **out)


CFG3_FULL_POINTS = (0, 6333, 12666, 18999)  # spread over the 19k cfg3 cache points


def _cfg3_full_one(i):
    """One bench-workload record (cfg3 room, n = 16384, step 0.1, n_inner 1, n_light 16) from
    the unmodified reference: estimate_moments' build_subdivision + assemble_moments and both
    make_record calls, with trace chunked per SURVEY.md §8d (per-ray identical)."""
    import volcache.transport as vt

    shim = _chunked_trace(vscene.trace, 16)
    for mod in (vscene, vr, vt):
        mod.trace = shim
    w = configs.cfg3()
    rs = ref_scene(w.scene)
    x = w.points[i]
    with Capture() as cap:
        sub = vs.build_subdivision(rs, x, n_angular=16384, march_step=0.1, rng_seed=vr._seed(2, 401, i), n_inner=1,
                                   n_light_samples=16)
    single, multiple, stats = vs.assemble_moments(sub, rs.medium)
    recs = [vcache.make_record(x, m, 0.05, rs.scale, rs.max_emission, anisotropic=True) for m in (single, multiple)]
    return dict(L=[single.L, multiple.L], grad=[single.grad, multiple.grad], hess=[single.hess, multiple.hess],
                stats=[stats["elements_evaluated"], stats["elements_dropped"], stats["star_vertices"]],
                adj=np.asarray(cap.dirs.adjacency, np.int32), s=cap.s, idx=np.asarray(cap.idx, np.int32),
                rec_value=[r.value for r in recs], rec_axes=[r.axes for r in recs], rec_radii=[r.radii for r in recs])


def gen_cfg3_full(procs=4):
    """Records of the bench workload itself from the reference: four cfg3
    points spread over the 19k, full n = 16384 with qhull's adjacency captured (the GPU test
    injects it).  ~35 min per record per core with the chunked brute-force trace."""
    import multiprocessing as mp
    import os

    os.environ.setdefault("OMP_NUM_THREADS", "1")
    w = configs.cfg3()
    with mp.get_context("fork").Pool(procs) as pool:
        res = pool.map(_cfg3_full_one, CFG3_FULL_POINTS)
    out = {k: np.array([r[k] for r in res]) for k in res[0]}
    dim, V, E, A = scene_arrays(w.scene)
    out.update(versions=VERSIONS, points=w.points[list(CFG3_FULL_POINTS)], index=np.array(CFG3_FULL_POINTS),
               cfg_seed=np.array(2), params=np.array([16384, 0.1, 1, 16, 0.0]),
               scene_digest=np.array([V.sum(), (V * V).sum(), E.sum(), float(len(V))]))
    np.savez_compressed(OUT / "rec_cfg3_full.npz", **out)
    print("wrote cfg3_full", flush=True)


def gen_cfg5_crop(src=REPO / "gpurun_out" / "cfg5_crop_records.npz"):
    """Reference frozen render of a 64×36 crop of the cfg5 frame (1920×1080 over the cfg3
    room, march step 0.01) from GPU-populated records (tools/cfg5_crop_fixture.py: the
    records near the crop's rays, a superset of every record covering a crop march point).
    The crop is a reference Camera whose rays are the full camera's rays of the crop pixels
    (render() itself is unchanged); trace is chunked (per-ray identical)."""
    import inspect
    import time

    z = np.load(src)
    r0, nr, c0, nc = (int(v) for v in z["crop"])
    sc3 = configs.cfg3_scene()
    sc = ref_scene(sc3)
    vscene_trace = vscene.trace
    shim = _chunked_trace(vscene_trace)
    for mod in (vscene, vr, __import__("volcache.transport", fromlist=["x"])):
        if hasattr(mod, "trace"):
            mod.trace = shim
    c = configs.cfg5_camera(1920, 1080)
    full = vr.Camera(position=c["position"], look_at=c["look_at"], up=c["up"], fov_degrees=c["fov"], width=1920,
                     height=1080)

    class CropCamera(vr.Camera):
        def rays(self, jitter):
            jf = np.full((full.height, full.width, 2), 0.5)
            jf[r0:r0 + nr, c0:c0 + nc] = jitter
            o, d = full.rays(jf)
            sel = (np.arange(r0, r0 + nr)[:, None] * full.width + np.arange(c0, c0 + nc)[None]).ravel()
            return o[sel], d[sel]

    crop = CropCamera(position=c["position"], look_at=c["look_at"], up=c["up"], fov_degrees=c["fov"], width=nc,
                      height=nr)
    st = vr.RenderSettings(mode="ours-aniso", epsilon=float(z["eps"]), spp=1, march_step=float(z["step"]),
                           n_angular=16384, seed=int(z["seed"]), frozen=True)
    cs = vr.CacheSet(sc, "ours-aniso")
    for name, cache in (("single", cs.single), ("multiple", cs.multiple)):
        for r in z[f"{name}_rows"]:
            cache.insert(vcache.CacheRecord(position=r[:3].copy(), value=r[3:6].copy(), grad=r[6:15].reshape(3, 3).copy(),
                                            axes=r[15:24].reshape(3, 3).copy(), radii=r[24:27].copy()))
    t0 = time.perf_counter()
    img, stats = vr.render(sc, crop, st, cache_set=cs)
    print("reference crop render", time.perf_counter() - t0, "s", {k: stats[k] for k in ("cache_hits",
                                                                                      "direct_evaluations")})
    assert stats["direct_evaluations"] == 0, "crop must be covered by the populated records"
    out = {"versions": VERSIONS, "crop": z["crop"], "eps": z["eps"], "step": z["step"], "seed": z["seed"],
           "single_rows": z["single_rows"], "multiple_rows": z["multiple_rows"],
           "single_index": z["single_index"], "multiple_index": z["multiple_index"],
           "pop_stats": z["pop_stats"], "image": img, "gpu_full_cache_crop": z["gpu_full_cache_crop"],
           "stats": np.array([stats["cache_hits"], stats["direct_evaluations"]])}
    np.savez_compressed(OUT / "cfg5_crop.npz", **out)
    for mod in (vscene, vr, __import__("volcache.transport", fromlist=["x"])):
        if hasattr(mod, "trace"):
            mod.trace = vscene_trace
    del inspect


def gen_path():
    """path_trace_radiance / fd_derivatives / render mode "path" through the reference
    (src/transport.py:318-391, src/renderer.py:337-346, :590-643)."""
    import volcache.transport as vt

    bundled = Path("/root/reference/pkg/scenes")
    pen = vscene.load_scene(bundled / "penumbra2d.json")
    box = vscene.load_scene(bundled / "box3d.json")
    box_refl = vscene.Scene(
        surfaces=tuple(vscene.Surface(vertices=s.vertices, emission=s.emission,
                                      albedo=(0.0 if s.is_emitter else 0.5)) for s in box.surfaces),
        medium=box.medium, bounds_min=box.bounds_min, bounds_max=box.bounds_max)
    out = {"versions": VERSIONS}
    out.update(scene_fields("pen_", pen))
    out.update(scene_fields("box_", box))
    out.update(scene_fields("boxr_", box_refl))
    cases = {  # name: (prefix, scene, x, n_samples, max_media_bounces, n_light, seed)
        "pen": ("pen_", pen, np.array([0.15, 0.6]), 70000, 2, 16, 5),
        "pen4": ("pen_", pen, np.array([0.5, 0.35]), 3000, 4, 8, 6),
        "box": ("box_", box, np.array([0.5, 0.5, 0.5]), 70000, 2, 8, 7),
        "boxr": ("boxr_", box_refl, np.array([0.3, 0.6, 0.4]), 5000, 3, 4, 8),
    }
    for name, (prefix, sc, x, n, mmb, nl, seed) in cases.items():
        s_, m_ = vt.path_trace_radiance(sc, x, n, max_media_bounces=mmb, rng_seed=seed, n_light_samples=nl)
        out[f"{name}_x"] = x
        out[f"{name}_params"] = np.array([n, mmb, nl, seed])
        out[f"{name}_J"] = np.array([s_, m_])
        out[f"{name}_prefix"] = np.array(prefix)
    fs, fm = vr.fd_derivatives(pen, np.array([0.3, 0.45]), h=0.02, n_samples=20000, seed=11, include_hessian=True)
    out["fd_pen"] = np.array([np.concatenate([e.value, e.grad.ravel(), e.hess.ravel()]) for e in (fs, fm)])
    fs, fm = vr.fd_derivatives(box, np.array([0.5, 0.4, 0.6]), h=0.03, n_samples=8000, seed=12, include_hessian=True,
                               n_light_samples=4)
    out["fd_box"] = np.array([np.concatenate([e.value, e.grad.ravel(), e.hess.ravel()]) for e in (fs, fm)])
    st = vr.RenderSettings(mode="path", path_samples_per_point=64, n_light_samples=4, seed=4)
    img, _ = vr.render(pen, vr.FieldGrid.for_scene(pen, 4, 3), st)
    out["render_field"] = img
    cam = vr.Camera(position=np.array([0.5, 0.5, 0.5]), look_at=np.array([0.5, 0.5, 1.0]),
                    up=np.array([0.0, 1.0, 0.0]), fov_degrees=60.0, width=3, height=2)
    st3 = vr.RenderSettings(mode="path", path_samples_per_point=32, n_light_samples=4, seed=5, spp=2, march_step=0.25)
    img3, _ = vr.render(box, cam, st3)
    out["render_camera"] = img3
    np.savez_compressed(OUT / "path.npz", **out)


def gen_grow():
    """Camera render with frozen=False (insertion during the march, src/renderer.py:361-368)."""
    bundled = Path("/root/reference/pkg/scenes")
    box = vscene.load_scene(bundled / "box3d.json")
    out = {"versions": VERSIONS}
    out.update(scene_fields("box_", box))
    cam = vr.Camera(position=np.array([0.5, 0.3, 0.05]), look_at=np.array([0.5, 0.5, 1.0]),
                    up=np.array([0.0, 1.0, 0.0]), fov_degrees=70.0, width=4, height=3)
    out["camera"] = np.concatenate([cam.position, cam.look_at, cam.up, [cam.fov_degrees, cam.width, cam.height]])
    for mode in ("baseline", "ours-aniso"):
        st = vr.RenderSettings(mode=mode, epsilon=0.1, march_step=0.2, n_angular=128, n_light_samples=4, seed=21,
                               spp=2, frozen=False)
        cs = vr.CacheSet(box, mode)
        img, stats = vr.render(box, cam, st, cache_set=cs)
        key = mode.replace("-", "_")
        out[f"{key}_image"] = img
        out[f"{key}_stats"] = np.array([stats["cache_hits"], stats["direct_evaluations"], len(cs.single),
                                        len(cs.multiple)])
        out.update(_records_fields(f"{key}_single", cs.single))
        out.update(_records_fields(f"{key}_multiple", cs.multiple))
    np.savez_compressed(OUT / "grow.npz", **out)


def gen_dropin():
    """Quadrature values the reference's estimator tests compare against
    (tests/test_subdivision.py:222-353: quadrature_radiance on the bundled scenes)."""
    import volcache.transport as vt

    sys.path.insert(0, "/root/reference/pkg/tests")
    from conftest import circle_scene  # the reference's own test scene helper

    bundled = Path("/root/reference/pkg/scenes")
    pen = vscene.load_scene(bundled / "penumbra2d.json")
    box = vscene.load_scene(bundled / "box3d.json")
    circ = circle_scene(n_sides=48, sigma_s=0.5, sigma_a=0.25)
    out = {"versions": VERSIONS}
    out.update(scene_fields("pen_", pen))
    out.update(scene_fields("box_", box))
    out.update(scene_fields("circ_", circ))
    out["q_pen"] = np.array(vt.quadrature_radiance(pen, np.array([0.15, 0.6]), n_angular=4096, n_dist=24,
                                                   n_secondary=64))
    out["q_circ"] = np.array(vt.quadrature_radiance(circ, np.array([0.5, 0.5]), n_angular=4096, n_dist=4,
                                                    n_secondary=4))
    out["q_box"] = np.array(vt.quadrature_radiance(box, np.array([0.5, 0.5, 0.5]), n_angular=3072, n_dist=6,
                                                   n_secondary=192))
    np.savez_compressed(OUT / "dropin.npz", **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["ff", "trace", "records", "make_record", "interp", "render", "populate", "io", "baseline", "path", "grow", "dropin"]
    if "ff" in which:
        gen_formfactors()
    if "trace" in which:
        gen_trace()
    if "records" in which:
        gen_records()
    for w in which:
        if w.startswith("records:"):  # e.g. records:room_refl
            gen_records(only=w.split(":", 1)[1].split(","))
    if "make_record" in which:
        gen_make_record()
    if "interp" in which:
        gen_interpolate()
    if "render" in which:
        gen_render()
    if "populate" in which:
        gen_populate()
    if "io" in which:
        gen_io()
    if "baseline" in which:
        gen_baseline()
    if "baseline_rng" in which:
        gen_baseline_rng()
    if "cfg3_full" in which:
        gen_cfg3_full()
    if "surface" in which:
        gen_surface()
    if "delta_lights" in which:
        gen_delta_lights()
    if "media_bounces" in which:
        gen_media_bounces()
    if "media_hg" in which:
        gen_media_hg()
    if "cfg5_crop" in which:
        gen_cfg5_crop()
    if "path" in which:
        gen_path()
    if "grow" in which:
        gen_grow()
    if "dropin" in which:
        gen_dropin()
