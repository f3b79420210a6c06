"""Pin the CPU oracle to the reference: oracle vs golden fixtures made by the reference.

CPU-only (no GPU marker).  Integer outputs (hit indices, adjacency, element counts)
must be identical; float outputs agree to ≤1e-12 relative, since the oracle
restates the reference's float64 arithmetic.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import REC_CASES, golden, golden_scene, rel_l2
from oracle import volcache_oracle as O


def test_formfactors_match_reference():
    z = golden("formfactors")
    ok, v, g, h = O.segment_ff(z["seg_x"], z["seg_y0"], z["seg_y1"])
    np.testing.assert_array_equal(ok, z["seg_ok"])
    np.testing.assert_allclose(v, z["seg_val"], rtol=1e-13, atol=0)
    np.testing.assert_allclose(g, z["seg_grad"], rtol=1e-12, atol=1e-300)
    np.testing.assert_allclose(h, z["seg_hess"], rtol=1e-11, atol=1e-300)
    ok, v, g, h = O.triangle_ff(z["tri_x"], z["tri_y1"], z["tri_y2"], z["tri_y3"])
    np.testing.assert_array_equal(ok, z["tri_ok"])
    np.testing.assert_allclose(v, z["tri_val"], rtol=1e-13, atol=0)
    np.testing.assert_allclose(g, z["tri_grad"], rtol=1e-12, atol=1e-300)
    np.testing.assert_allclose(h, z["tri_hess"], rtol=1e-11, atol=1e-300)
    assert (~z["seg_ok"]).sum() >= 8 and (~z["tri_ok"]).sum() >= 8  # degenerate cases present


@pytest.mark.parametrize("name", ["c1", "c2", "room"])
def test_trace_matches_reference(name):
    z = golden("trace")
    ps = O.pack(golden_scene(z, f"{name}_"))
    s, idx = O.trace_or_bounds(ps, z[f"{name}_o"], z[f"{name}_d"])
    np.testing.assert_array_equal(idx, z[f"{name}_idx"])
    np.testing.assert_array_equal(s, z[f"{name}_s"])


@pytest.mark.parametrize("case", REC_CASES)
def test_records_match_reference(case):
    z = golden(f"rec_{case}")
    ps = O.pack(golden_scene(z))
    n, step, n_inner, n_light, canon = z["params"]
    seed = int(z["cfg_seed"])
    for i, x in enumerate(z["points"]):
        inject = z["adj"][i] if canon else None
        rb = O.build_record(ps, x, int(n), float(step), O.seed_seq(seed, 401, i), int(n_inner),
                            int(n_light), adjacency=inject)
        np.testing.assert_array_equal(rb.adjacency, z["adj"][i])
        np.testing.assert_array_equal(rb.idx, z["idx"][i])
        np.testing.assert_array_equal(rb.s, z["s"][i])
        np.testing.assert_array_equal(rb.dirs, z["dirs"][i])
        st = rb.stats
        assert [st["elements_evaluated"], st["elements_dropped"], st["star_vertices"]] == z["stats"][i].tolist()
        for k in range(2):
            assert rel_l2(rb.L[k], z["L"][i][k]) <= 1e-12
            assert rel_l2(rb.grad[k], z["grad"][i][k]) <= 1e-11
            assert rel_l2(rb.hess[k], z["hess"][i][k]) <= 1e-10
            rec = O.make_record(x, rb.L[k], rb.grad[k], rb.hess[k], 0.05, ps.scale, ps.max_emission)
            np.testing.assert_allclose(rec.radii, z["rec_radii"][i][k], rtol=1e-9)
            q = rec.axes @ np.diag(rec.radii**-2.0) @ rec.axes.T
            qz = z["rec_axes"][i][k] @ np.diag(z["rec_radii"][i][k] ** -2.0) @ z["rec_axes"][i][k].T
            assert rel_l2(q, qz) <= 1e-8


def test_media_bounces_oracle_matches_reference_shim():
    """The ≤ B-bounce media-radiance extension in the oracle (gather_mean_bounces) against
    the reference's build_subdivision + assemble_moments run with a gather written from the
    reference's own primitives (make_goldens.py gen_media_bounces, B = 4)."""
    z = golden("rec_media_bounces")
    ps = O.pack(golden_scene(z))
    n, step, n_inner, n_light, B = z["params"]
    for i, x in enumerate(z["points"]):
        rb = O.build_record(ps, x, int(n), float(step), O.seed_seq(int(z["cfg_seed"]), 401, i), int(n_inner),
                            int(n_light), adjacency=z["adj"][i], media_bounces=int(B))
        st = rb.stats
        assert [st["elements_evaluated"], st["elements_dropped"], st["star_vertices"]] == z["stats"][i].tolist()
        for k in range(2):
            assert rel_l2(rb.L[k], z["L"][i][k]) <= 1e-12
            assert rel_l2(rb.grad[k], z["grad"][i][k]) <= 1e-11
            assert rel_l2(rb.hess[k], z["hess"][i][k]) <= 1e-10
    # the extension changes only the multiple-scattering moments
    rb1 = O.build_record(ps, z["points"][0], int(n), float(step), O.seed_seq(int(z["cfg_seed"]), 401, 0),
                         adjacency=z["adj"][0])
    assert rel_l2(rb1.L[0], z["L"][0][0]) <= 1e-12 and rel_l2(rb1.L[1], z["L"][0][1]) > 1e-3


def test_surface_radiance_matches_reference():
    """The oracle's surface_radiance (direct lighting with shadow rays) on the reflective
    small room against the reference's surface_radiance_batch (tests/golden/surface.npz)."""
    from paper_1805_09258_b200 import configs

    z = golden("surface")
    ps = O.pack(configs.cfg3_scene(n_spheres=4, level=1, wall_albedo=0.5))
    lo = O.surface_radiance(ps, z["small_idx"], z["small_points"], z["small_dirs"], 16)
    np.testing.assert_allclose(lo, z["small_lo"], rtol=1e-12, atol=1e-15)


def test_media_hg_oracle_matches_reference_shim():
    """The Henyey–Greenstein extension (g = 0.5 at the media sample and at every further media
    event, 4 events per gather path) in the oracle against the reference's build_subdivision +
    assemble_moments with the gather rebuilt from its primitives (gen_media_hg)."""
    z = golden("rec_media_hg")
    ps = O.pack(golden_scene(z))
    n, step, n_inner, n_light, B, g = z["params"]
    for i, x in enumerate(z["points"]):
        rb = O.build_record(ps, x, int(n), float(step), O.seed_seq(int(z["cfg_seed"]), 401, i), int(n_inner),
                            int(n_light), adjacency=z["adj"][i], media_bounces=int(B), hg_g=float(g))
        assert [rb.stats["elements_evaluated"], rb.stats["elements_dropped"], rb.stats["star_vertices"]] == \
            z["stats"][i].tolist()
        for k in range(2):
            assert rel_l2(rb.L[k], z["L"][i][k]) <= 1e-12
            assert rel_l2(rb.grad[k], z["grad"][i][k]) <= 1e-11
            assert rel_l2(rb.hess[k], z["hess"][i][k]) <= 1e-10


DELTA_CASES = ("d2", "refl", "portal", "hg")


@pytest.mark.parametrize("case", DELTA_CASES)
def test_delta_lights_oracle_matches_reference_shim(case):
    """The delta-light extension (point and directional lights on reflective surfaces, at every
    media sample and at the cache point; with HG and further media events in `hg`) in the
    oracle against the reference's build_subdivision + assemble_moments with direct_lighting
    and the gather extended through the reference's own trace / bounds_exit (gen_delta_lights)."""
    z = golden("rec_delta_lights")
    ps = O.pack(golden_scene(z, case + "_"))
    assert len(ps.lights) >= 1
    n, step, n_inner, n_light, B, g, seed = z[case + "_params"]
    for i, x in enumerate(z[case + "_points"]):
        rb = O.build_record(ps, x, int(n), float(step), O.seed_seq(int(seed), 401, i), int(n_inner), int(n_light),
                            adjacency=z[case + "_adj"][i], media_bounces=int(B), hg_g=float(g))
        assert [rb.stats["elements_evaluated"], rb.stats["elements_dropped"], rb.stats["star_vertices"]] == \
            z[case + "_stats"][i].tolist()
        for k in range(2):
            assert rel_l2(rb.L[k], z[case + "_L"][i][k]) <= 1e-12
            assert rel_l2(rb.grad[k], z[case + "_grad"][i][k]) <= 1e-11
            assert rel_l2(rb.hess[k], z[case + "_hess"][i][k]) <= 1e-10


def test_delta_lights_off_is_the_reference():
    """No lights → every delta-light hook is inert (the reference's estimator exactly)."""
    z = golden("rec_delta_lights")
    sc = golden_scene(z, "portal_")
    ps = O.pack(sc)
    ps0 = O.pack(golden_scene({k: z[k] for k in z.files if not k.endswith("_lights")}, "portal_"))
    assert len(ps0.lights) == 0 and len(ps.lights) == 1
    n, step, n_inner, n_light, B, g, seed = z["portal_params"]
    x = z["portal_points"][0]
    a = O.build_record(ps, x, int(n), float(step), O.seed_seq(int(seed), 401, 0), adjacency=z["portal_adj"][0])
    b = O.build_record(ps0, x, int(n), float(step), O.seed_seq(int(seed), 401, 0), adjacency=z["portal_adj"][0])
    assert np.all(a.L[1] > b.L[1]) and np.all(a.L[0] > b.L[0])  # the lamp adds light everywhere
    np.testing.assert_array_equal(a.idx, b.idx)


def test_make_record_edge_cases():
    z = golden("make_record")
    for j in range(int(z["n_cases"])):
        dim = int(z[f"c{j}_dim"])
        for aniso in (True, False):
            for max_em in (10, 0):
                key = f"c{j}_{int(aniso)}_{max_em}"
                rec = O.make_record(z[f"c{j}_x"], z[f"c{j}_L"], z[f"c{j}_g"], z[f"c{j}_H"], 0.05,
                                    float(np.sqrt(dim)), float(max_em), anisotropic=aniso)
                np.testing.assert_allclose(rec.radii, z[key + "_radii"], rtol=1e-10)
                q = rec.axes @ np.diag(rec.radii**-2.0) @ rec.axes.T
                qz = z[key + "_axes"] @ np.diag(z[key + "_radii"] ** -2.0) @ z[key + "_axes"].T
                assert rel_l2(q, qz) <= 1e-8, (j, aniso, max_em)


@pytest.mark.parametrize("dim", [2, 3])
def test_interpolate_matches_reference(dim):
    z = golden("interpolate")
    recs = [O.Record(*a) for a in zip(z[f"d{dim}_pos"], z[f"d{dim}_value"], z[f"d{dim}_grad"],
                                      z[f"d{dim}_axes"], z[f"d{dim}_radii"])]
    cache = O.Cache(recs)
    for x, J, c in zip(z[f"d{dim}_q"], z[f"d{dim}_J"], z[f"d{dim}_count"]):
        assert len(cache.query(x)) == c
        v = O.interpolate(cache, x)
        if np.isnan(J[0]):
            assert v is None
        else:
            np.testing.assert_allclose(v, J, rtol=1e-13)


def test_render_matches_reference():
    z = golden("render")
    ps = O.pack(golden_scene(z))
    caches = []
    for kind in ("single", "multiple"):
        caches.append(O.Cache([O.Record(*a) for a in zip(z[f"{kind}_pos"], z[f"{kind}_value"], z[f"{kind}_grad"],
                                                        z[f"{kind}_axes"], z[f"{kind}_radii"])]))
    eps, spp, step, n_ang, seed, n_inner, n_light = z["settings"]
    c = z["camera"]
    cam = dict(position=c[0:3], look_at=c[3:6], up=c[6:9], fov=c[9], width=int(c[10]), height=int(c[11]))
    prm = O.RenderParams(epsilon=eps, spp=int(spp), march_step=step, n_angular=int(n_ang), seed=int(seed),
                         n_inner=int(n_inner), n_light_samples=int(n_light))
    img, stats = O.render_camera(ps, cam, caches[0], caches[1], prm)
    np.testing.assert_allclose(img.reshape(z["image"].shape), z["image"], rtol=1e-12, atol=1e-14)
    assert stats["cache_hits"] == int(z["stats"][0])
    assert stats["direct_evaluations"] == int(z["stats"][1])


def _prm(v):
    eps, step, n, nl, seed, n_inner, spp, frozen, iso = v
    return O.RenderParams(epsilon=float(eps), spp=int(spp), march_step=float(step), n_angular=int(n),
                          seed=int(seed), n_light_samples=int(nl), n_inner=int(n_inner), anisotropic=not iso)


def _field(z, prefix, nx, ny):
    return {"kind": "field", "nx": nx, "ny": ny, "bmin": z[prefix + "bmin"], "bmax": z[prefix + "bmax"]}


def _camera_target(v):
    return {"kind": "camera", "position": v[0:3], "look_at": v[3:6], "up": v[6:9], "fov": float(v[9]),
            "width": int(v[10]), "height": int(v[11])}


def _rows(cache):
    return np.array([np.concatenate([r.position, r.value, r.grad.ravel(), r.axes.ravel(), r.radii])
                     for r in cache.records]).reshape(len(cache.records), -1)


def _assert_rows(got, want, d):
    assert got.shape == want.shape
    np.testing.assert_array_equal(got[:, :d], want[:, :d])
    assert rel_l2(got[:, d:], want[:, d:]) <= 1e-9


@pytest.mark.parametrize("name,prefix,nx,ny", [("simple6", "simple_", 6, 6), ("pen8_tight", "pen_", 8, 8),
                                               ("pen16_iso", "pen_", 16, 12)])
def test_populate_field_matches_reference(name, prefix, nx, ny):
    z = golden("populate")
    ps = O.pack(golden_scene(z, prefix))
    s, m, n = O.populate_cache(ps, _field(z, prefix, nx, ny), _prm(z[f"{name}_settings"]))
    assert [n, len(s.records), len(m.records)] == z[f"{name}_stats"].tolist()
    _assert_rows(_rows(s), z[f"{name}_single"], 2)
    _assert_rows(_rows(m), z[f"{name}_multiple"], 2)


@pytest.mark.parametrize("name", ["box32", "box108"])
def test_populate_camera_matches_reference(name):
    z = golden("populate")
    ps = O.pack(golden_scene(z, "box_"))
    s, m, n = O.populate_cache(ps, _camera_target(z[f"{name}_camera"]), _prm(z[f"{name}_settings"]))
    assert [n, len(s.records), len(m.records)] == z[f"{name}_stats"].tolist()
    _assert_rows(_rows(s), z[f"{name}_single"], 3)
    _assert_rows(_rows(m), z[f"{name}_multiple"], 3)


def test_render_field_matches_reference():
    z = golden("populate")
    ps = O.pack(golden_scene(z, "pen_"))
    prm = _prm(z["render_pen65_settings"])
    tgt = _field(z, "pen_", 6, 5)
    s, m, _ = O.populate_cache(ps, tgt, prm)
    img, st = O.render_field(ps, tgt, s, m, prm)
    assert [st["cache_hits"], st["direct_evaluations"], len(s.records) + len(m.records)] == \
        z["render_pen65_stats"].tolist()
    np.testing.assert_allclose(img, z["render_pen65_image"], rtol=1e-11)
    ps = O.pack(golden_scene(z, "simple_"))
    prm = _prm(z["render_frozen_settings"])
    s, m = O.Cache(), O.Cache()
    img, st = O.render_field(ps, _field(z, "simple_", 3, 3), s, m, prm, frozen=True)
    assert [st["cache_hits"], st["direct_evaluations"], 0] == z["render_frozen_stats"].tolist()
    np.testing.assert_allclose(img, z["render_frozen_image"], rtol=1e-11)
    prm = _prm(z["render_grow_settings"])
    img, st = O.render_field(ps, _field(z, "simple_", 6, 6), s, m, prm, frozen=False)
    assert [st["cache_hits"], st["direct_evaluations"], len(s.records) + len(m.records)] == \
        z["render_grow_stats"].tolist()
    np.testing.assert_allclose(img, z["render_grow_image"], rtol=1e-11)
    _assert_rows(_rows(s), z["render_grow_single"], 2)


def test_render_camera_growing_matches_reference():
    """frozen=False camera render (insertion during the march) vs the reference's run."""
    z = golden("grow")
    ps = O.pack(golden_scene(z, "box_"))
    v = z["camera"]
    cam = dict(position=v[0:3], look_at=v[3:6], up=v[6:9], fov=float(v[9]), width=int(v[10]), height=int(v[11]))
    prm = O.RenderParams(epsilon=0.1, spp=2, march_step=0.2, n_angular=128, seed=21, n_light_samples=4)
    s, m = O.Cache(), O.Cache()
    img, st = O.render_camera(ps, cam, s, m, prm, frozen=False)
    assert [st["cache_hits"], st["direct_evaluations"], len(s.records), len(m.records)] == \
        z["ours_aniso_stats"].tolist()
    np.testing.assert_allclose(img.reshape(z["ours_aniso_image"].shape), z["ours_aniso_image"], rtol=1e-11)
    _assert_rows(_rows(s), z["ours_aniso_single"], 3)
