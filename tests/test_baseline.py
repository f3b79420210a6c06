"""GPU occlusion-unaware baseline against the reference's own outputs.

tests/golden/baseline.npz (make_goldens.py gen_baseline) holds baseline_estimate values,
gradients and per-sample luminance/gradient norms, make_baseline_record radii,
log_space_interpolate answers and a baseline-mode populate + render for a FieldGrid
and a camera (src/subdivision.py:416-521, src/cache.py:190-394, src/renderer.py:233-244).
The baseline uses no triangulation, so 3D matches the reference directly.
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden, golden_scene, rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield


@pytest.mark.parametrize("name", ["pen", "pen3", "box", "boxr"])
def test_baseline_estimate_matches_reference(name):
    from paper_1805_09258_b200.baseline import baseline_estimate, make_baseline_record
    from paper_1805_09258_b200.renderer import _seed

    z = golden("baseline")
    sc = golden_scene(z, str(z[f"{name}_prefix"]))
    n, mmb, nl = (int(v) for v in z[f"{name}_params"])
    for i, x in enumerate(z[f"{name}_points"]):
        s, m = baseline_estimate(sc, x, n_angular=n, rng_seed=_seed(17, 401, i), max_media_bounces=mmb,
                                 n_light_samples=nl)
        for k, est in enumerate((s, m)):
            assert est.kind == ("single", "multiple")[k]
            assert rel_l2(est.value, z[f"{name}_value"][i][k], floor=1e-300) <= 1e-9
            assert rel_l2(est.grad, z[f"{name}_grad"][i][k], floor=1e-300) <= 1e-9
            np.testing.assert_allclose(est.sample_values, z[f"{name}_svals"][i][k], rtol=1e-9, atol=1e-300)
            np.testing.assert_allclose(est.sample_grad_norms, z[f"{name}_snorms"][i][k], rtol=1e-9, atol=1e-300)
            rec = make_baseline_record(x, est, sc.scale, 0.7)
            np.testing.assert_allclose(rec.radius, z[f"{name}_radius"][i][k], rtol=1e-9)


def test_baseline_batch_records_match_single_calls():
    from paper_1805_09258_b200.baseline import baseline_estimate, baseline_records_batch, make_baseline_record
    from paper_1805_09258_b200.records import seed_words
    from paper_1805_09258_b200.renderer import _seed

    z = golden("baseline")
    sc = golden_scene(z, "box_")
    pts = z["box_points"]
    words = seed_words(17, 401, np.arange(len(pts)))
    est, rec = baseline_records_batch(sc, pts, words, n_angular=1024, max_media_bounces=2, n_light_samples=8,
                                      alpha=0.7)
    for i, x in enumerate(pts):
        s, m = baseline_estimate(sc, x, n_angular=1024, rng_seed=_seed(17, 401, i), max_media_bounces=2,
                                 n_light_samples=8)
        for k, e in enumerate((s, m)):
            np.testing.assert_array_equal(est[i, k, :3], e.value)
            r = make_baseline_record(x, e, sc.scale, 0.7)
            np.testing.assert_allclose(rec[i, k, -1], r.radius, rtol=1e-12)
            np.testing.assert_array_equal(rec[i, k, :3], x)


def test_log_space_interpolate_matches_reference():
    from paper_1805_09258_b200.baseline import log_space_interpolate
    from paper_1805_09258_b200.cache import RadianceCache
    from paper_1805_09258_b200.io import BaselineRecord

    z = golden("baseline")
    cache = RadianceCache(np.zeros(3), np.ones(3))
    for r in z["log_records"]:
        cache.insert(BaselineRecord(position=r[:3], value=r[3:6], grad=r[6:15].reshape(3, 3), radius=float(r[15])))
    J, cnt = cache.interpolate_many(z["log_q"], log_space=True)
    want = z["log_J"]
    none = np.isnan(want[:, 0])
    assert none.any() and (~none).any()
    np.testing.assert_array_equal(np.isnan(J[:, 0]), none)
    np.testing.assert_allclose(J[~none], want[~none], rtol=1e-12, atol=1e-300)
    v = log_space_interpolate(cache, z["log_q"][0])
    assert (v is None) == bool(none[0])


def _rows_equal(got, want, d):
    assert got.shape == want.shape, (got.shape, want.shape)
    if len(want):
        np.testing.assert_array_equal(got[:, :d], want[:, :d])
        assert rel_l2(got[:, d:], want[:, d:]) <= 1e-9


def test_baseline_mode_field_populate_and_render():
    from paper_1805_09258_b200.renderer import FieldGrid, RenderSettings, populate_cache, render

    z = golden("baseline")
    sc = golden_scene(z, "pen_")
    st = RenderSettings(mode="baseline", epsilon=0.05, march_step=0.1, n_angular=64, n_light_samples=4, seed=3,
                        baseline_alpha=0.8)
    grid = FieldGrid.for_scene(sc, 8, 6)
    cs, pst = populate_cache(sc, grid, st)
    _rows_equal(cs.single.packed(), z["bpop_single"], 2)
    _rows_equal(cs.multiple.packed(), z["bpop_multiple"], 2)
    img, rst = render(sc, grid, st, cache_set=cs)
    assert [pst["points_marched"], pst["records_single"], pst["records_multiple"], rst["cache_hits"],
            rst["direct_evaluations"]] == z["bpop_stats"].tolist()
    assert rel_l2(img, z["bpop_image"]) <= 1e-9


def test_baseline_mode_camera_populate_and_render():
    from paper_1805_09258_b200.renderer import Camera, RenderSettings, populate_cache, render

    z = golden("baseline")
    sc = golden_scene(z, "box_")
    v = z["bcam_camera"]
    cam = Camera(position=v[0:3], look_at=v[3:6], up=v[6:9], fov_degrees=float(v[9]), width=int(v[10]),
                 height=int(v[11]))
    st = RenderSettings(mode="baseline", epsilon=0.1, march_step=0.1, n_angular=256, n_light_samples=4, seed=9, spp=1)
    cs, pst = populate_cache(sc, cam, st)
    _rows_equal(cs.single.packed(), z["bcam_single"], 3)
    _rows_equal(cs.multiple.packed(), z["bcam_multiple"], 3)
    img, rst = render(sc, cam, st, cache_set=cs)
    assert [pst["points_marched"], pst["records_single"], pst["records_multiple"], rst["cache_hits"],
            rst["direct_evaluations"]] == z["bcam_stats"].tolist()
    assert rel_l2(img, z["bcam_image"]) <= 1e-9
