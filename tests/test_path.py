"""GPU path-traced reference and FD derivative oracle vs the reference.

tests/golden/path.npz (make_goldens.py gen_path) holds path_trace_radiance values (with
> 2^16 samples, i.e. several of the reference's draw chunks), fd_derivatives with the
Hessian stencil, and render mode "path" images for a FieldGrid and a jittered camera
(src/transport.py:318-391, src/renderer.py:337-346, :590-643).  Same streams, same
draws: agreement is to float64 rounding of the sums.
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


@pytest.mark.parametrize("name", ["pen", "pen4", "box", "boxr"])
def test_path_trace_matches_reference(name):
    from paper_1805_09258_b200.path import path_trace_radiance

    z = golden("path")
    sc = golden_scene(z, str(z[f"{name}_prefix"]))
    n, mmb, nl, seed = (int(v) for v in z[f"{name}_params"])
    s, m = path_trace_radiance(sc, z[f"{name}_x"], n, max_media_bounces=mmb, rng_seed=seed, n_light_samples=nl)
    assert rel_l2(s, z[f"{name}_J"][0], floor=1e-300) <= 1e-10
    assert rel_l2(m, z[f"{name}_J"][1], floor=1e-300) <= 1e-10


def test_path_trace_validation_and_determinism():
    from paper_1805_09258_b200.path import path_trace_radiance

    z = golden("path")
    sc = golden_scene(z, "pen_")
    with pytest.raises(ValueError):
        path_trace_radiance(sc, np.array([1.5, 0.5]), 128, rng_seed=0)
    a = path_trace_radiance(sc, np.array([0.3, 0.5]), 4096, rng_seed=5)
    b = path_trace_radiance(sc, np.array([0.3, 0.5]), 4096, rng_seed=5)
    c = path_trace_radiance(sc, np.array([0.3, 0.5]), 4096, rng_seed=6)
    np.testing.assert_array_equal(a[0], b[0])
    assert not np.array_equal(a[0], c[0])


@pytest.mark.parametrize("name,prefix,x,h,n,seed,nl", [
    ("fd_pen", "pen_", [0.3, 0.45], 0.02, 20000, 11, 16),
    ("fd_box", "box_", [0.5, 0.4, 0.6], 0.03, 8000, 12, 4)])
def test_fd_derivatives_match_reference(name, prefix, x, h, n, seed, nl):
    from paper_1805_09258_b200.path import fd_derivatives

    z = golden("path")
    sc = golden_scene(z, prefix)
    s, m = fd_derivatives(sc, np.array(x), h=h, n_samples=n, seed=seed, include_hessian=True, n_light_samples=nl)
    d = len(x)
    for k, e in enumerate((s, m)):
        want = z[name][k]
        assert rel_l2(e.value, want[:3], floor=1e-300) <= 1e-10
        # differences of nearly equal CRN sums: compare at the scale of the values
        scale = max(np.abs(want[:3]).max(), 1e-300)
        np.testing.assert_allclose(e.grad.ravel(), want[3:3 + 3 * d], rtol=0, atol=1e-9 * scale / h)
        np.testing.assert_allclose(e.hess.ravel(), want[3 + 3 * d:], rtol=0, atol=1e-9 * scale / h ** 2)


def test_render_path_mode_matches_reference():
    from paper_1805_09258_b200.renderer import Camera, FieldGrid, RenderSettings, render

    z = golden("path")
    sc = golden_scene(z, "pen_")
    st = RenderSettings(mode="path", path_samples_per_point=64, n_light_samples=4, seed=4)
    img, stats = render(sc, FieldGrid.for_scene(sc, 4, 3), st)
    assert "populate" not in stats and stats["mode"] == "path"
    assert rel_l2(img, z["render_field"]) <= 1e-10
    box = golden_scene(z, "box_")
    cam = Camera(position=np.array([0.5, 0.5, 0.5]), look_at=np.array([0.5, 0.5, 1.0]), up=np.array([0.0, 1.0, 0.0]),
                 fov_degrees=60.0, width=3, height=2)
    st3 = RenderSettings(mode="path", path_samples_per_point=32, n_light_samples=4, seed=5, spp=2, march_step=0.25)
    img3, _ = render(box, cam, st3)
    assert rel_l2(img3, z["render_camera"]) <= 1e-10
