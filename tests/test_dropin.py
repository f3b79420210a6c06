"""The reference's estimator-level tests, run against the B200 drop-ins.

Mirrors tests/test_subdivision.py:192-353 of the reference (dataclass shapes,
determinism, agreement with the deterministic quadrature, derivatives against
common-random-number path-traced finite differences, the occlusion-unaware baseline)
with the same inputs and tolerances.  The quadrature values were computed by the
reference itself (tests/golden/dropin.npz, make_goldens.py gen_dropin); the FD
oracle runs on the device (paper_1805_09258_b200.path, checked against the reference's
own fd_derivatives in test_path.py).
"""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden, golden_scene

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    yield


def rel_error(approx, exact, floor=0.0):  # volcache.oracles.rel_error (src/oracles.py:82-89)
    approx, exact = np.asarray(approx, float), np.asarray(exact, float)
    denom = max(float(np.linalg.norm(exact)), floor)
    if denom == 0.0:
        return float(np.linalg.norm(approx - exact))
    return float(np.linalg.norm(approx - exact)) / denom


@pytest.fixture(scope="module")
def z():
    return golden("dropin")


@pytest.fixture(scope="module")
def pen(z):
    return golden_scene(z, "pen_")


@pytest.fixture(scope="module")
def simple():
    return golden_scene(golden("populate"), "simple_")


def test_moments_dataclass_shape(pen):
    from paper_1805_09258_b200 import Moments, estimate_moments

    single, multiple = estimate_moments(pen, np.array([0.2, 0.7]), n_angular=128, march_step=0.1, rng_seed=0)
    assert isinstance(single, Moments) and single.kind == "single"
    assert isinstance(multiple, Moments) and multiple.kind == "multiple"
    assert single.dim == 2 and single.L.shape == (3,) and single.grad.shape == (3, 2)
    assert single.hess.shape == (3, 2, 2)
    for c in range(3):
        np.testing.assert_allclose(single.hess[c], single.hess[c].T)
        np.testing.assert_allclose(multiple.hess[c], multiple.hess[c].T)


def test_estimate_deterministic_by_seed(pen):
    from paper_1805_09258_b200 import estimate_moments

    x = np.array([0.3, 0.5])
    a = estimate_moments(pen, x, n_angular=128, rng_seed=9)
    b = estimate_moments(pen, x, n_angular=128, rng_seed=9)
    c = estimate_moments(pen, x, n_angular=128, rng_seed=10)
    np.testing.assert_array_equal(a[0].L, b[0].L)
    np.testing.assert_array_equal(a[0].grad, b[0].grad)
    assert not np.array_equal(a[0].L, c[0].L)


def test_values_match_quadrature(z, pen):
    from paper_1805_09258_b200 import estimate_moments

    q_single, q_multiple = z["q_pen"]
    single, multiple = estimate_moments(pen, np.array([0.15, 0.6]), n_angular=2048, march_step=0.05, rng_seed=3,
                                        n_inner=4)
    assert rel_error(single.L, q_single, floor=1e-9) < 0.05
    assert rel_error(multiple.L, q_multiple, floor=1e-9) < 0.05


def test_enclosure_value(z):
    from paper_1805_09258_b200 import estimate_moments

    circ = golden_scene(z, "circ_")
    q_single, _ = z["q_circ"]
    single, _ = estimate_moments(circ, np.array([0.5, 0.5]), n_angular=1024, march_step=1.0, rng_seed=0)
    assert rel_error(single.L, q_single, floor=1e-12) < 0.01


def test_gradient_and_hessian_match_path_fd(pen):
    from paper_1805_09258_b200 import estimate_moments, fd_derivatives

    x = np.array([0.15, 0.6])
    fd_single, _ = fd_derivatives(pen, x, h=0.01, n_samples=1_000_000, seed=11)
    single, _ = estimate_moments(pen, x, n_angular=4096, march_step=0.05, rng_seed=3)
    assert rel_error(single.grad, fd_single.grad, floor=1e-9) < 0.05
    fd_h, _ = fd_derivatives(pen, x, h=0.02, n_samples=2_000_000, seed=11, include_hessian=True)
    assert rel_error(single.hess, fd_h.hess, floor=1e-6) < 0.25


def test_multiple_gradient_matches_path_fd(pen):
    from paper_1805_09258_b200 import estimate_moments, fd_derivatives

    x = np.array([0.15, 0.6])
    _, fd_multiple = fd_derivatives(pen, x, h=0.01, n_samples=1_000_000, seed=11)
    _, multiple = estimate_moments(pen, x, n_angular=8192, march_step=0.02, rng_seed=3, n_inner=8)
    assert rel_error(multiple.grad, fd_multiple.grad, floor=1e-9) < 0.25


def test_baseline_estimate_shapes(pen):
    from paper_1805_09258_b200 import BaselineEstimate, baseline_estimate

    single, multiple = baseline_estimate(pen, np.array([0.3, 0.5]), n_angular=512, rng_seed=0)
    for est, kind in ((single, "single"), (multiple, "multiple")):
        assert isinstance(est, BaselineEstimate) and est.kind == kind
        assert est.value.shape == (3,) and est.grad.shape == (3, 2)
        assert est.sample_values.shape == (512,) and est.sample_grad_norms.shape == (512,)
        assert np.all(est.sample_values >= 0.0) and np.all(est.sample_grad_norms >= 0.0)


def test_baseline_value_matches_quadrature(z, pen):
    from paper_1805_09258_b200 import baseline_estimate

    q_single, q_multiple = z["q_pen"]
    single, multiple = baseline_estimate(pen, np.array([0.15, 0.6]), n_angular=8192, rng_seed=4)
    assert rel_error(single.value, q_single, floor=1e-9) < 0.03
    assert rel_error(multiple.value, q_multiple, floor=1e-9) < 0.25


def test_baseline_gradient_fine_without_occlusion(simple):
    from paper_1805_09258_b200 import baseline_estimate, fd_derivatives

    x = np.array([0.5, 0.4])
    fd_single, _ = fd_derivatives(simple, x, h=0.01, n_samples=500_000, seed=2)
    single, _ = baseline_estimate(simple, x, n_angular=8192, rng_seed=5)
    assert rel_error(single.grad, fd_single.grad, floor=1e-9) < 0.1


def test_baseline_gradient_wrong_in_penumbra(pen):
    from paper_1805_09258_b200 import baseline_estimate, estimate_moments, fd_derivatives

    x = np.array([0.3, 0.45])
    fd_single, _ = fd_derivatives(pen, x, h=0.01, n_samples=1_000_000, seed=7)
    base_single, _ = baseline_estimate(pen, x, n_angular=4096, rng_seed=6)
    sub_single, _ = estimate_moments(pen, x, n_angular=4096, march_step=0.05, rng_seed=6)
    assert rel_error(sub_single.grad, fd_single.grad, floor=1e-9) < rel_error(base_single.grad, fd_single.grad,
                                                                              floor=1e-9)


def test_occlusion_unaware_gradient_wrapper(pen):
    from paper_1805_09258_b200 import baseline_estimate, occlusion_unaware_gradient

    g1, g2 = occlusion_unaware_gradient(pen, np.array([0.3, 0.5]), n_angular=256, rng_seed=0)
    single, multiple = baseline_estimate(pen, np.array([0.3, 0.5]), n_angular=256, rng_seed=0)
    np.testing.assert_array_equal(g1, single.grad)
    np.testing.assert_array_equal(g2, multiple.grad)


def test_3d_moments_match_quadrature(z):
    from paper_1805_09258_b200 import estimate_moments

    box = golden_scene(z, "box_")
    single, multiple = estimate_moments(box, np.array([0.5, 0.5, 0.5]), n_angular=3072, march_step=0.25,
                                        rng_seed=0, n_inner=2)
    q_single, q_multiple = z["q_box"]
    assert rel_error(single.L, q_single, floor=1e-9) < 0.05
    assert rel_error(multiple.L, q_multiple, floor=1e-9) < 0.2
    assert single.grad.shape == (3, 3)
    for c in range(3):
        np.testing.assert_allclose(single.hess[c], single.hess[c].T)
    # ceiling emitter above: the vertical gradient dominates and points up
    assert single.grad[0, 2] > abs(single.grad[0, 0])
    assert single.grad[0, 2] > abs(single.grad[0, 1])
