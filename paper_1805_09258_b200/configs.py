"""Synthetic workloads for BASELINE.json's configs (parity variants).

The reference supports area emitters only and isotropic homogeneous media
(SPEC.md:13, :149), so each config is expressed as its reference-runnable
"parity variant": point/directional lights become small emissive quads or
window portals, HG phase becomes isotropic, and multiple scattering is the
reference's one extra bounce (src/subdivision.py:175-195).  Cache points are
`default_rng(cfg_seed).uniform(bounds_min, bounds_max, (N, d))` and per-record
streams are `SeedSequence([cfg_seed, 401, i])` (src/renderer.py:278-279, :317).
No public dataset is involved; the paper's Statues scene is replaced by the
seeded icosphere "window room".
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .scene import Medium, Scene, Surface, directional_light, point_light


@dataclass(frozen=True)
class Workload:
    name: str
    scene: Scene
    points: np.ndarray  # (N, d)
    seed: int  # cfg seed: record i uses SeedSequence([seed, 401, i])
    n_angular: int
    march_step: float
    n_inner: int = 1
    n_light_samples: int = 16
    epsilon: float = 0.05
    media_bounces: int = 1  # extension: media events per gather path (1 = the reference)
    hg_g: float = 0.0  # extension: Henyey-Greenstein g of the media scattering events (0 = the reference)

    @property
    def dim(self) -> int:
        return self.points.shape[1]


def _seg(a, b, emission=0.0, albedo=0.0):
    return Surface(vertices=np.array([a, b], float), emission=emission, albedo=albedo)


def _tri(a, b, c, emission=0.0, albedo=0.0):
    return Surface(vertices=np.array([a, b, c], float), emission=emission, albedo=albedo)


def _quad(p0, p1, p2, p3, emission=0.0, albedo=0.0):
    return [_tri(p0, p1, p2, emission, albedo), _tri(p0, p2, p3, emission, albedo)]


def _rect_2d(x0, y0, x1, y1, emission=0.0, albedo=0.0):
    c = [(x0, y0), (x1, y0), (x1, y1), (x0, y1)]
    return [_seg(c[i], c[(i + 1) % 4], emission, albedo) for i in range(4)]


def _box_3d(center, side, emission=0.0, albedo=0.0):
    h = 0.5 * side
    cx, cy, cz = center
    v = np.array(
        [[cx + sx * h, cy + sy * h, cz + sz * h] for sx in (-1, 1) for sy in (-1, 1) for sz in (-1, 1)]
    )
    faces = [(0, 1, 3, 2), (4, 6, 7, 5), (0, 4, 5, 1), (2, 3, 7, 6), (0, 2, 6, 4), (1, 5, 7, 3)]
    out = []
    for a, b, c, d in faces:
        out += _quad(v[a], v[b], v[c], v[d], emission, albedo)
    return out


def icosphere(level: int):
    """Unit icosphere: 20·4^level triangles (level 3 → 1280)."""
    t = (1.0 + 5.0 ** 0.5) / 2.0
    verts = [
        (-1, t, 0), (1, t, 0), (-1, -t, 0), (1, -t, 0),
        (0, -1, t), (0, 1, t), (0, -1, -t), (0, 1, -t),
        (t, 0, -1), (t, 0, 1), (-t, 0, -1), (-t, 0, 1),
    ]
    verts = [np.array(v, float) / np.linalg.norm(v) for v in verts]
    faces = [
        (0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11),
        (1, 5, 9), (5, 11, 4), (11, 10, 2), (10, 7, 6), (7, 1, 8),
        (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8), (3, 8, 9),
        (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1),
    ]
    for _ in range(level):
        cache = {}

        def mid(a, b):
            key = (min(a, b), max(a, b))
            if key not in cache:
                m = verts[a] + verts[b]
                verts.append(m / np.linalg.norm(m))
                cache[key] = len(verts) - 1
            return cache[key]

        nf = []
        for a, b, c in faces:
            ab, bc, ca = mid(a, b), mid(b, c), mid(c, a)
            nf += [(a, ab, ca), (b, bc, ab), (c, ca, bc), (ab, bc, ca)]
        faces = nf
    return np.array(verts), np.array(faces)


# ---------------------------------------------------------------------------
# Config 1: 2D flatland, point light → small emissive square
# ---------------------------------------------------------------------------


def cfg1_scene() -> Scene:
    side = 0.02
    c = (0.2, 0.8)
    light = _rect_2d(c[0] - side / 2, c[1] - side / 2, c[0] + side / 2, c[1] + side / 2,
                     emission=1.0 / side)
    occ = _rect_2d(0.4, 0.45, 0.6, 0.55)
    return Scene(tuple(light + occ), Medium(0.5, 0.1), np.zeros(2), np.ones(2))


def cfg1_spec_scene(occluder_albedo: float = 0.0) -> Scene:
    """Extension: cfg1 as BASELINE.json states it — a point light (intensity 1) instead of the
    emissive square (delta lights are not in the reference)."""
    occ = _rect_2d(0.4, 0.45, 0.6, 0.55, albedo=occluder_albedo)
    return Scene(tuple(occ), Medium(0.5, 0.1), np.zeros(2), np.ones(2),
                 lights=np.array([point_light((0.2, 0.8), 1.0)]))


def cfg1(n_points: int = 256, march_step: float = 4.0) -> Workload:
    sc = cfg1_scene()
    pts = np.random.default_rng(0).uniform(sc.bounds_min, sc.bounds_max, (n_points, 2))
    return Workload("cfg1-flatland-2d", sc, pts, 0, 1024, march_step)


# ---------------------------------------------------------------------------
# Config 2: 3D single occluder, point light → 0.1×0.1 emissive quad
# ---------------------------------------------------------------------------


def cfg2_scene() -> Scene:
    y = 0.95
    h = 0.05
    light = _quad((0.5 - h, y, 0.5 - h), (0.5 + h, y, 0.5 - h), (0.5 + h, y, 0.5 + h),
                  (0.5 - h, y, 0.5 + h), emission=100.0)
    cube = _box_3d((0.5, 0.6, 0.5), 0.2)
    return Scene(tuple(light + cube), Medium(0.8, 0.2), np.zeros(3), np.ones(3))


def cfg2_spec_scene() -> Scene:
    """Extension: cfg2 as BASELINE.json states it — an isotropic point light at (0.5, 0.95, 0.5)
    (used with hg_g = 0.3)."""
    cube = _box_3d((0.5, 0.6, 0.5), 0.2)
    return Scene(tuple(cube), Medium(0.8, 0.2), np.zeros(3), np.ones(3),
                 lights=np.array([point_light((0.5, 0.95, 0.5), 1.0)]))


def cfg2(n_points: int = 4096, march_step: float = 4.0) -> Workload:
    sc = cfg2_scene()
    pts = np.random.default_rng(1).uniform(sc.bounds_min, sc.bounds_max, (n_points, 3))
    return Workload("cfg2-single-occluder-3d", sc, pts, 1, 4096, march_step)


# ---------------------------------------------------------------------------
# Config 3: 4×3×4 window room with 40 level-3 icospheres (~51k triangles)
# ---------------------------------------------------------------------------

ROOM = np.array([4.0, 3.0, 4.0])
WINDOW_EMISSION = np.array([20.0, 19.0, 17.0])


SUN_TOWARD = np.array([-1.0, 0.55, 0.2])  # cfg3-spec: from the room toward the distant light
SUN_IRRADIANCE = np.array([20.0, 19.0, 17.0])


def _window_wall(emission, open_windows=False):
    """Wall x = 0 tiled by a cut grid; the 8 window cells (2 rows × 4) are emissive portals
    (or, open_windows, cut-outs a directional light shines through)."""
    zc = [0.6, 1.53, 2.47, 3.4]
    yc = [1.0, 2.1]
    hw, hh = 0.3, 0.35
    zs = sorted({0.0, ROOM[2], *[z - hw for z in zc], *[z + hw for z in zc]})
    ys = sorted({0.0, ROOM[1], *[y - hh for y in yc], *[y + hh for y in yc]})
    out = []
    for j in range(len(ys) - 1):
        for i in range(len(zs) - 1):
            z0, z1, y0, y1 = zs[i], zs[i + 1], ys[j], ys[j + 1]
            zm, ym = 0.5 * (z0 + z1), 0.5 * (y0 + y1)
            win = any(abs(zm - z) < hw for z in zc) and any(abs(ym - y) < hh for y in yc)
            if win and open_windows:
                continue
            out += _quad((0, y0, z0), (0, y0, z1), (0, y1, z1), (0, y1, z0),
                         emission=emission if win else 0.0)
    return out


def cfg3_scene(n_spheres: int = 40, level: int = 3, seed: int = 2, wall_albedo: float = 0.0,
               open_windows: bool = False, lights=(), window_emission=WINDOW_EMISSION,
               medium: Medium | None = None) -> Scene:
    """open_windows / lights: the delta-light extension (cfg3 as BASELINE.json states it: window
    cut-outs lit by a distant directional light); the default is the reference-runnable parity
    variant with emissive portals."""
    X, Y, Z = ROOM
    walls = _window_wall(window_emission, open_windows)
    walls += _quad((X, 0, 0), (X, 3, 0), (X, 3, Z), (X, 0, Z), albedo=wall_albedo)  # far side
    walls += _quad((0, 0, 0), (X, 0, 0), (X, 0, Z), (0, 0, Z), albedo=wall_albedo)  # floor
    walls += _quad((0, Y, 0), (0, Y, Z), (X, Y, Z), (X, Y, 0), albedo=wall_albedo)  # ceiling
    walls += _quad((0, 0, 0), (0, Y, 0), (X, Y, 0), (X, 0, 0), albedo=wall_albedo)  # z = 0
    walls += _quad((0, 0, Z), (X, 0, Z), (X, Y, Z), (0, Y, Z), albedo=wall_albedo)  # z = 4
    rng = np.random.default_rng(seed)
    V, F = icosphere(level)
    spheres = []
    for _ in range(n_spheres):
        c = rng.uniform([0.6, 0.4, 0.5], [3.6, 2.6, 3.5])
        r = rng.uniform(0.12, 0.3)
        P = c[None] + r * V
        spheres += [_tri(P[a], P[b], P[d]) for a, b, d in F]
    return Scene(tuple(walls + spheres), medium or Medium(0.27, 0.03), np.zeros(3), ROOM.copy(),
                 lights=np.asarray(lights, float).reshape(-1, 8))


def cfg3_spec_scene(n_spheres: int = 40, level: int = 3, wall_albedo: float = 0.0) -> Scene:
    """Extension: cfg3 as BASELINE.json states it — open window cut-outs and a distant
    directional light (used with hg_g = 0.5 and media_bounces = 4)."""
    return cfg3_scene(n_spheres, level, wall_albedo=wall_albedo, open_windows=True,
                      lights=[directional_light(SUN_TOWARD, SUN_IRRADIANCE)])


def cfg3(n_points: int = 19000, n_spheres: int = 40, level: int = 3, n_angular: int = 16384,
         march_step: float = 0.1) -> Workload:
    sc = cfg3_scene(n_spheres, level)
    pts = np.random.default_rng(2).uniform(sc.bounds_min, sc.bounds_max, (n_points, 3))
    return Workload("cfg3-window-room-3d", sc, pts, 2, n_angular, march_step)


# ---------------------------------------------------------------------------
# Config 4 stand-in: cfg3's occluders, 8 seeded point lights, homogeneous medium
# ---------------------------------------------------------------------------


def cfg4_standin_scene(n_spheres: int = 40, level: int = 3) -> Scene:
    """Extension, and only a stand-in: BASELINE.json's cfg4 is a heterogeneous Perlin medium
    with ratio tracking, which the method does not cover (its ∇T, HT assume a constant σt;
    PAPER.md:603 lists heterogeneous media as future work).  This keeps cfg4's geometry
    (cfg3's occluder set, no emissive windows) and its 8 seeded point lights (seed 3) in a
    homogeneous medium at the grid's nominal mean density: σt = 2 (max 4 × mean 0.5),
    albedo 0.85."""
    rng = np.random.default_rng(3)
    pos = rng.uniform([0.4, 0.4, 0.4], ROOM - 0.4, (8, 3))
    lights = [point_light(p, (3.0, 3.0, 3.0)) for p in pos]
    return cfg3_scene(n_spheres, level, lights=lights, window_emission=0.0, medium=Medium(1.7, 0.3))


def cfg4_standin(n_points: int = 32000, n_angular: int = 16384, march_step: float = 0.1) -> Workload:
    sc = cfg4_standin_scene()
    pts = np.random.default_rng(3).uniform(sc.bounds_min, sc.bounds_max, (n_points, 3))
    return Workload("cfg4-standin-homogeneous+8-point-lights", sc, pts, 3, n_angular, march_step)


# ---------------------------------------------------------------------------
# Config 5: camera over the config-3 room
# ---------------------------------------------------------------------------


def cfg5_camera(width: int = 1920, height: int = 1080) -> dict:
    return {
        "position": np.array([2.0, 1.5, 0.2]),
        "look_at": np.array([2.0, 1.5, 4.0]),
        "up": np.array([0.0, 1.0, 0.0]),
        "fov": 60.0,
        "width": width,
        "height": height,
    }


CONFIGS = {"cfg1": cfg1, "cfg2": cfg2, "cfg3": cfg3}
