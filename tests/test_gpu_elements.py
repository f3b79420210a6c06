"""Device element math against the reference's own outputs, edge cases included.

* vc_form_factors (the float64 ff_segment / ff_triangle of the record build, and the float32
  3D element path) on tests/golden/formfactors.npz: 256 segment and 256 triangle rows from
  ff_segment_derivs_batch / ff_triangle_derivs_batch, with thin, vertex-coincident and
  coplanar (degenerate) rows (src/formfactor.py:23-30, :99-106, :306).
* vc_make_records (k_make_record: closed-form eigen, Jacobi fallback, radii) on every case
  of tests/golden/make_record.npz: random, zero, rank-1, repeated, negative-definite, tiny
  and diagonal Hessians in 2D and 3D, anisotropic and isotropic, max_emission 10 and 0
  (src/cache.py:59-91, :146-189; src/numerics.py:127-166).
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden, rel_l2

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.set_device(0)
    yield


def _ff(dim, x, verts, precision=0):
    from paper_1805_09258_b200 import _lib

    x = np.ascontiguousarray(x, float)
    verts = np.ascontiguousarray(verts, float)
    m = x.shape[0]
    ok = np.zeros(m, np.uint8)
    v = np.zeros(m)
    g = np.zeros((m, dim))
    h = np.zeros((m, dim, dim))
    _lib.check(_lib.lib().vc_form_factors(dim, m, _lib.ptr(x), _lib.ptr(verts), precision, _lib.VC_MEM_HOST,
                                          _lib.ptr(ok), _lib.ptr(v), _lib.ptr(g), _lib.ptr(h), None))
    return ok.astype(bool), v, g, h


def _rel_rows(a, b, floor):
    a = a.reshape(len(a), -1)
    b = b.reshape(len(b), -1)
    return np.linalg.norm(a - b, axis=1) / np.maximum(np.linalg.norm(b, axis=1), floor)


def test_segment_form_factors_match_reference():
    z = golden("formfactors")
    ok, v, g, h = _ff(2, z["seg_x"], np.stack([z["seg_y0"], z["seg_y1"]], axis=1))
    np.testing.assert_array_equal(ok, z["seg_ok"])
    assert (~ok).sum() >= 8  # the degenerate rows are exercised
    assert np.all(v[~ok] == 0) and np.all(g[~ok] == 0) and np.all(h[~ok] == 0)
    assert np.max(_rel_rows(v, z["seg_val"], 1e-300)[ok]) <= 1e-9
    assert np.max(_rel_rows(g, z["seg_grad"], 1e-300)[ok]) <= 1e-9
    assert np.max(_rel_rows(h, z["seg_hess"], 1e-300)[ok]) <= 1e-9


@pytest.mark.parametrize("precision", [0, 1])
def test_triangle_form_factors_match_reference(precision):
    z = golden("formfactors")
    verts = np.stack([z["tri_y1"], z["tri_y2"], z["tri_y3"]], axis=1)
    ok, v, g, h = _ff(3, z["tri_x"], verts, precision)
    np.testing.assert_array_equal(ok, z["tri_ok"])  # ok-mask decided in float64 on both paths
    assert (~ok).sum() >= 8
    assert np.all(v[~ok] == 0) and np.all(g[~ok] == 0) and np.all(h[~ok] == 0)
    ev = _rel_rows(v, z["tri_val"], 1e-300)[ok]
    eg = _rel_rows(g, z["tri_grad"], 1e-300)[ok]
    eh = _rel_rows(h, z["tri_hess"], 1e-300)[ok]
    if precision == 0:
        assert max(ev.max(), eg.max(), eh.max()) <= 1e-9
    else:
        # float32 element math: per element, relative to the element's own magnitude; the
        # per-record gates (L 1e-4, ∇/H 1e-3) are asserted on whole records elsewhere
        assert np.median(ev) <= 1e-5 and np.median(eg) <= 1e-4 and np.median(eh) <= 1e-4
        assert np.quantile(eh, 0.95) <= 1e-3


def test_form_factor_argument_errors():
    from paper_1805_09258_b200 import _lib

    with pytest.raises(ValueError):
        _lib.check(_lib.lib().vc_form_factors(4, 1, None, None, 0, _lib.VC_MEM_HOST, None, None, None, None, None))
    with pytest.raises(ValueError):
        _ff(2, np.zeros((1, 2)), np.zeros((1, 2, 2)), precision=1)
    ok, v, _, _ = _ff(3, np.zeros((0, 3)), np.zeros((0, 3, 3)))
    assert ok.size == 0


def test_make_record_edge_cases_on_device():
    from paper_1805_09258_b200.records import make_records, moment_size

    z = golden("make_record")
    worst_r = worst_q = 0.0
    for j in range(int(z["n_cases"])):
        d = int(z[f"c{j}_dim"])
        mom = np.zeros((1, 2, moment_size(d)))
        mom[0, :, :3] = z[f"c{j}_L"]
        mom[0, :, 3:3 + 3 * d] = z[f"c{j}_g"].ravel()
        mom[0, :, 3 + 3 * d:] = z[f"c{j}_H"].ravel()
        for aniso in (True, False):
            for max_em in (10, 0):
                key = f"c{j}_{int(aniso)}_{max_em}"
                rec = make_records(z[f"c{j}_x"][None], mom, 0.05, float(np.sqrt(d)), float(max_em), aniso)[0, 0]
                axes = rec[d + 3 + 3 * d:d + 3 + 3 * d + d * d].reshape(d, d)
                radii = rec[-d:]
                zr, za = z[key + "_radii"], z[key + "_axes"]
                np.testing.assert_allclose(radii, zr, rtol=1e-10, err_msg=key)
                q = axes @ np.diag(radii ** -2.0) @ axes.T
                qz = za @ np.diag(zr ** -2.0) @ za.T
                eq = rel_l2(q, qz)
                assert eq <= 1e-8, (key, eq)
                np.testing.assert_array_equal(rec[:d], z[f"c{j}_x"])
                np.testing.assert_array_equal(rec[d:d + 3], z[f"c{j}_L"])
                worst_r = max(worst_r, float(np.max(np.abs(radii - zr) / zr)))
                worst_q = max(worst_q, eq)
    print("make_record edge cases: worst radius rel", worst_r, "worst quadratic form rel", worst_q)
