"""GPU populate_cache / field render / camera render against the reference's own runs.

tests/golden/populate.npz holds the record sets, images and stats the reference
produced (make_goldens.py gen_populate, src/renderer.py:282-484).  The device engine
must insert the same records in the same order: positions bit-exact (they are march
points), values ≤ 1e-4 and gradients / axes·radii ≤ 1e-3 relative, stats exact.
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


def _settings(v):
    from paper_1805_09258_b200.renderer import RenderSettings

    eps, step, n, nl, seed, n_inner, spp, frozen, iso = v
    return RenderSettings(mode="ours-iso" if iso else "ours-aniso", epsilon=float(eps), march_step=float(step),
                          n_angular=int(n), n_light_samples=int(nl), seed=int(seed), n_inner=int(n_inner),
                          spp=int(spp), frozen=bool(frozen))


def _camera(v):
    from paper_1805_09258_b200.renderer import Camera

    return Camera(position=v[0:3], look_at=v[3:6], up=v[6:9], fov_degrees=float(v[9]), width=int(v[10]),
                  height=int(v[11]))


def _quadratic_forms(rows, d):
    ax = rows[:, d + 3 + 3 * d: d + 3 + 3 * d + d * d].reshape(-1, d, d)
    rad = rows[:, -d:]
    return np.einsum("nij,nj,nkj->nik", ax, 1.0 / rad ** 2, ax)


def _same_records(got, want, d):
    assert got.shape == want.shape, (got.shape, want.shape)
    if len(want) == 0:
        return
    np.testing.assert_array_equal(got[:, :d], want[:, :d])  # insertion order and positions
    assert rel_l2(got[:, d:d + 3], want[:, d:d + 3]) <= 1e-4
    assert rel_l2(got[:, d + 3:d + 3 + 3 * d], want[:, d + 3:d + 3 + 3 * d]) <= 1e-3
    qa, qb = _quadratic_forms(got, d), _quadratic_forms(want, d)
    for a, b in zip(qa, qb):
        assert rel_l2(a, b) <= 1e-3


SCENES = {"simple6": "simple_", "pen8_tight": "pen_", "pen8_loose": "pen_", "pen16_iso": "pen_", "pen64": "pen_"}
FIELD = {"simple6": (6, 6), "pen8_tight": (8, 8), "pen8_loose": (8, 8), "pen16_iso": (16, 12), "pen64": (64, 48)}


@pytest.mark.parametrize("name", list(FIELD))
def test_populate_field_matches_reference(name):
    from paper_1805_09258_b200.renderer import FieldGrid, populate_cache

    z = golden("populate")
    sc = golden_scene(z, SCENES[name])
    st = _settings(z[f"{name}_settings"])
    nx, ny = FIELD[name]
    cs, stats = populate_cache(sc, FieldGrid.for_scene(sc, nx, ny), st)
    want = z[f"{name}_stats"]
    assert stats["points_marched"] == int(want[0])
    assert (stats["records_single"], stats["records_multiple"]) == (int(want[1]), int(want[2]))
    assert stats["records"] == cs.record_count
    _same_records(cs.single.packed(), z[f"{name}_single"], 2)
    _same_records(cs.multiple.packed(), z[f"{name}_multiple"], 2)
    # every marched point is covered afterwards (src/renderer.py:320-324)
    grid = FieldGrid.for_scene(sc, nx, ny)
    pts = grid.centers.reshape(-1, 2)
    for c in (cs.single, cs.multiple):
        _, cnt = c.interpolate_many(pts)
        assert np.all(cnt > 0)


@pytest.mark.parametrize("window,lookahead", [(1, 1), (3, 5), (7, 64), (2048, 1 << 20)])
def test_populate_independent_of_speculation(window, lookahead):
    """Window size and lookahead change only how much is speculated, never the result."""
    from paper_1805_09258_b200.renderer import FieldGrid, populate_cache

    z = golden("populate")
    sc = golden_scene(z, "pen_")
    st = _settings(z["pen8_tight_settings"])
    cs, stats = populate_cache(sc, FieldGrid.for_scene(sc, 8, 8), st, window=window, lookahead=lookahead)
    ref, _ = populate_cache(sc, FieldGrid.for_scene(sc, 8, 8), st)
    np.testing.assert_array_equal(cs.single.packed(), ref.single.packed())
    np.testing.assert_array_equal(cs.multiple.packed(), ref.multiple.packed())
    _same_records(cs.single.packed(), z["pen8_tight_single"], 2)


def _oracle_rows(cache):
    return np.array([np.concatenate([r.position, r.value, r.grad.ravel(), r.axes.ravel(), r.radii])
                     for r in cache.records]).reshape(len(cache.records), -1)


@pytest.mark.parametrize("name", ["box32", "box108", "box3224"])
def test_populate_camera_matches_oracle(name):
    """3D camera populate vs the oracle's sequential loop with the same (GPU) triangulations.

    In 3D the multiple-scattering estimate depends on the vertex order of each spherical
    Delaunay triangle (the representative media sample, src/subdivision.py:175-195); qhull's
    order is an artefact of its insertion sequence, so the device triangulation's order is
    injected into the oracle (which is itself pinned to the reference's populate runs in
    test_oracle_golden.py).  Counts and positions then match the sequential loop exactly.
    """
    from oracle import volcache_oracle as O
    from paper_1805_09258_b200 import inspect_record
    from paper_1805_09258_b200.renderer import populate_cache

    z = golden("populate")
    sc = golden_scene(z, "box_")
    st = _settings(z[f"{name}_settings"])
    cam = _camera(z[f"{name}_camera"])
    cs, stats = populate_cache(sc, cam, st)
    center = 0.5 * (sc.bounds_min + sc.bounds_max)

    def gpu_adjacency(seed):  # the triangulation depends only on the record's stream
        return inspect_record(sc, center, rng_seed=seed, n_angular=st.n_angular, march_step=st.march_step)["tris"]

    v = z[f"{name}_camera"]
    tgt = {"kind": "camera", "position": v[0:3], "look_at": v[3:6], "up": v[6:9], "fov": float(v[9]),
           "width": int(v[10]), "height": int(v[11])}
    prm = O.RenderParams(epsilon=st.epsilon, spp=1, march_step=st.march_step, n_angular=st.n_angular, seed=st.seed,
                         n_light_samples=st.n_light_samples, n_inner=st.n_inner)
    s, m, n = O.populate_cache(O.pack(sc), tgt, prm, adjacency_fn=gpu_adjacency)
    assert stats["points_marched"] == n == int(z[f"{name}_stats"][0])
    _same_records(cs.single.packed(), _oracle_rows(s), 3)
    _same_records(cs.multiple.packed(), _oracle_rows(m), 3)
    # single scattering does not involve the vertex order: equal to the reference's own run
    _same_records(cs.single.packed(), z[f"{name}_single"], 3)


def test_populate_room_matches_reference_render_golden():
    """The window room of render.npz: populate on the device, compare the reference's records."""
    from paper_1805_09258_b200.renderer import Camera, RenderSettings, populate_cache

    z = golden("render")
    sc = golden_scene(z)
    eps, spp, step, n_ang, seed, n_inner, n_light = z["settings"]
    cam = z["camera"]
    camera = Camera(position=cam[0:3], look_at=cam[3:6], up=cam[6:9], fov_degrees=float(cam[9]),
                    width=int(cam[10]), height=int(cam[11]))
    st = RenderSettings(mode="ours-aniso", epsilon=float(eps), spp=int(spp), march_step=float(step),
                        n_angular=int(n_ang), seed=int(seed), n_inner=int(n_inner), n_light_samples=int(n_light))
    cs, stats = populate_cache(sc, camera, st)
    assert stats["points_marched"] == int(z["stats"][2])
    want = np.concatenate([z["single_pos"], z["single_value"], z["single_grad"].reshape(-1, 9),
                           z["single_axes"].reshape(-1, 9), z["single_radii"]], axis=1)
    _same_records(cs.single.packed(), want, 3)


def test_render_field_default_matches_reference():
    from paper_1805_09258_b200.renderer import FieldGrid, render

    z = golden("populate")
    sc = golden_scene(z, "pen_")
    st = _settings(z["render_pen65_settings"])
    img, stats = render(sc, FieldGrid.for_scene(sc, 6, 5), st)
    want = z["render_pen65_stats"]
    assert (stats["cache_hits"], stats["direct_evaluations"], stats["records"]) == tuple(int(v) for v in want)
    assert "populate" in stats
    assert rel_l2(img, z["render_pen65_image"]) <= 1e-4


def test_render_field_frozen_empty_cache():
    from paper_1805_09258_b200.renderer import CacheSet, FieldGrid, render

    z = golden("populate")
    sc = golden_scene(z, "simple_")
    st = _settings(z["render_frozen_settings"])
    empty = CacheSet(sc, "ours-aniso")
    img, stats = render(sc, FieldGrid.for_scene(sc, 3, 3), st, cache_set=empty)
    assert empty.record_count == 0
    assert (stats["cache_hits"], stats["direct_evaluations"]) == (0, 9)
    assert rel_l2(img, z["render_frozen_image"]) <= 1e-4


def test_render_field_growing_cache():
    """frozen=False: misses insert in scanline order, later cells read the blend back."""
    from paper_1805_09258_b200.renderer import CacheSet, FieldGrid, render

    z = golden("populate")
    sc = golden_scene(z, "simple_")
    st = _settings(z["render_grow_settings"])
    growing = CacheSet(sc, "ours-aniso")
    img, stats = render(sc, FieldGrid.for_scene(sc, 6, 6), st, cache_set=growing)
    want = z["render_grow_stats"]
    assert (stats["cache_hits"], stats["direct_evaluations"], growing.record_count) == tuple(int(v) for v in want)
    _same_records(growing.single.packed(), z["render_grow_single"], 2)
    _same_records(growing.multiple.packed(), z["render_grow_multiple"], 2)
    assert rel_l2(img, z["render_grow_image"]) <= 1e-4


def test_populate_validation():
    from paper_1805_09258_b200.renderer import (Camera, CacheSet, FieldGrid, RenderSettings, populate_cache,
                                                render)

    z = golden("populate")
    sc2 = golden_scene(z, "simple_")
    sc3 = golden_scene(z, "box_")
    with pytest.raises(ValueError):
        populate_cache(sc2, FieldGrid.for_scene(sc2, 4, 4), RenderSettings(mode="path"))
    with pytest.raises(ValueError):
        render(sc3, FieldGrid(np.zeros(2), np.ones(2), 2, 2), RenderSettings())
    cam = Camera(position=np.array([0.5, 0.5, 0.5]), look_at=np.array([0.5, 0.5, 1.0]), up=np.array([0.0, 1.0, 0.0]),
                 fov_degrees=60.0, width=2, height=2)
    with pytest.raises(ValueError):
        render(sc2, cam, RenderSettings())
    with pytest.raises(TypeError):
        render(sc2, "not a target", RenderSettings())
    with pytest.raises(ValueError):
        CacheSet(sc2, "path")


def test_render_camera_growing_baseline_matches_reference():
    """frozen=False camera render in baseline mode (no triangulation): equal to the reference."""
    from paper_1805_09258_b200.renderer import CacheSet, RenderSettings, render

    z = golden("grow")
    sc = golden_scene(z, "box_")
    cam = _camera(z["camera"])
    st = RenderSettings(mode="baseline", epsilon=0.1, march_step=0.2, n_angular=128, n_light_samples=4, seed=21,
                        spp=2, frozen=False)
    cs = CacheSet(sc, "baseline")
    img, stats = render(sc, cam, st, cache_set=cs)
    assert [stats["cache_hits"], stats["direct_evaluations"], len(cs.single), len(cs.multiple)] == \
        z["baseline_stats"].tolist()
    np.testing.assert_array_equal(cs.single.packed()[:, :3], z["baseline_single"][:, :3])
    assert rel_l2(cs.multiple.packed(), z["baseline_multiple"]) <= 1e-9
    assert rel_l2(img, z["baseline_image"]) <= 1e-9


def test_render_camera_growing_matches_oracle():
    """frozen=False camera render, subdivision records: vs the oracle with the GPU triangulations."""
    from oracle import volcache_oracle as O
    from paper_1805_09258_b200 import inspect_record
    from paper_1805_09258_b200.renderer import CacheSet, RenderSettings, render

    z = golden("grow")
    sc = golden_scene(z, "box_")
    cam = _camera(z["camera"])
    st = RenderSettings(mode="ours-aniso", epsilon=0.1, march_step=0.2, n_angular=128, n_light_samples=4, seed=21,
                        spp=2, frozen=False)
    cs = CacheSet(sc, "ours-aniso")
    img, stats = render(sc, cam, st, cache_set=cs)
    center = 0.5 * (sc.bounds_min + sc.bounds_max)

    def gpu_adjacency(seed):
        return inspect_record(sc, center, rng_seed=seed, n_angular=128, march_step=0.2)["tris"]

    v = z["camera"]
    ocam = dict(position=v[0:3], look_at=v[3:6], up=v[6:9], fov=float(v[9]), width=int(v[10]), height=int(v[11]))
    prm = O.RenderParams(epsilon=0.1, spp=2, march_step=0.2, n_angular=128, seed=21, n_light_samples=4)
    s, m = O.Cache(), O.Cache()
    oimg, ost = O.render_camera(O.pack(sc), ocam, s, m, prm, adjacency_fn=gpu_adjacency, frozen=False)
    assert (stats["cache_hits"], stats["direct_evaluations"]) == (ost["cache_hits"], ost["direct_evaluations"])
    _same_records(cs.single.packed(), _oracle_rows(s), 3)
    _same_records(cs.multiple.packed(), _oracle_rows(m), 3)
    assert rel_l2(img, oimg.reshape(img.shape)) <= 1e-4


def test_populate_edge_cases():
    """Empty marches (camera looking away from the medium), a 1×1 field, a zero-step camera."""
    from paper_1805_09258_b200.renderer import Camera, FieldGrid, RenderSettings, populate_cache, render

    z = golden("populate")
    box = golden_scene(z, "box_")
    st = RenderSettings(mode="ours-aniso", epsilon=0.2, march_step=0.25, n_angular=128, n_light_samples=4, spp=1)
    away = Camera(position=np.array([0.5, 0.5, -2.0]), look_at=np.array([0.5, 0.5, -3.0]),
                  up=np.array([0.0, 1.0, 0.0]), fov_degrees=30.0, width=4, height=3)
    cs, stats = populate_cache(box, away, st)
    assert stats["points_marched"] == 0 and cs.record_count == 0
    img, rst = render(box, away, st, cache_set=cs)
    assert np.all(img == 0.0) and rst["direct_evaluations"] == 0
    sc2 = golden_scene(z, "simple_")
    st2 = RenderSettings(mode="ours-aniso", epsilon=0.05, march_step=0.1, n_angular=64, n_light_samples=4, seed=3)
    cs, stats = populate_cache(sc2, FieldGrid.for_scene(sc2, 1, 1), st2)
    assert stats["points_marched"] == 1 and stats["records_single"] == 1 and stats["records_multiple"] == 1
    np.testing.assert_array_equal(cs.single.packed()[0, :2], [0.5, 0.5])


def test_render_rows_stitch_to_full_render():
    """Row slabs (the unit of the row-sharded multi-GPU render) equal the full frozen render's
    rows bit for bit, and the hit / evaluation counts add up."""
    from paper_1805_09258_b200.renderer import RenderSettings, populate_cache, render, render_rows

    z = golden("render")
    sc = golden_scene(z)
    eps, spp, step, n_ang, seed, n_inner, n_light = z["settings"]
    camera = _camera(z["camera"])
    st = RenderSettings(mode="ours-aniso", epsilon=float(eps), spp=int(spp), march_step=float(step),
                        n_angular=int(n_ang), seed=int(seed), n_inner=int(n_inner), n_light_samples=int(n_light),
                        frozen=True)
    cs, _ = populate_cache(sc, camera, st)
    full, fst = render(sc, camera, st, cs)
    H = camera.height
    cuts = [0, 1, H // 2, H]
    hits = evals = 0
    for a, b in zip(cuts[:-1], cuts[1:]):
        slab, s = render_rows(sc, camera, st, cs, a, b - a)
        np.testing.assert_array_equal(slab, full[a:b])
        hits += s["cache_hits"]
        evals += s["direct_evaluations"]
    assert (hits, evals) == (fst["cache_hits"], fst["direct_evaluations"])
    empty, s0 = render_rows(sc, camera, st, cs, H, 0)
    assert empty.shape == (0, camera.width, 3) and s0["cache_hits"] == 0
    with pytest.raises(ValueError):
        render_rows(sc, camera, st, cs, H - 1, 2)


def test_render_sharded_nccl_world1_matches_render():
    """dist.render_sharded + broadcast_cache_set over NCCL (one rank on this GPU): the
    gathered image and counts equal the single-process frozen render."""
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    code = r'''
import os, sys, socket, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from conftest import golden, golden_scene
from paper_1805_09258_b200.renderer import Camera, RenderSettings, populate_cache, render
from paper_1805_09258_b200 import dist as vdist
s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1)
z = golden("render"); sc = golden_scene(z)
eps, spp, step, n_ang, seed, n_inner, n_light = z["settings"]; v = z["camera"]
cam = Camera(position=v[0:3], look_at=v[3:6], up=v[6:9], fov_degrees=float(v[9]), width=int(v[10]), height=int(v[11]))
st = RenderSettings(mode="ours-aniso", epsilon=float(eps), spp=int(spp), march_step=float(step), n_angular=int(n_ang),
                    seed=int(seed), n_inner=int(n_inner), n_light_samples=int(n_light), frozen=True)
cs, _ = populate_cache(sc, cam, st)
full, fst = render(sc, cam, st, cs)
vdist.broadcast_cache_set(cs)
img, s2 = vdist.render_sharded(sc, cam, st, cs)
np.testing.assert_array_equal(img, full)
assert (s2["cache_hits"], s2["direct_evaluations"]) == (fst["cache_hits"], fst["direct_evaluations"])
dist.destroy_process_group()
print("sharded ok")
'''
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "sharded ok" in r.stdout


def test_populate_sharded_nccl_world1_matches_populate():
    """dist.populate_sharded over NCCL (one rank on this GPU): every speculative wave goes
    through the engine's build hook (shard → device build → all-gather → resolve) and the
    caches equal the plain populate record for record, with the same engine statistics."""
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parents[1]
    code = r'''
import os, sys, socket, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from conftest import golden, golden_scene
from paper_1805_09258_b200.renderer import Camera, RenderSettings, populate_cache
from paper_1805_09258_b200 import dist as vdist
s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1)
z = golden("render"); sc = golden_scene(z)
eps, spp, step, n_ang, seed, n_inner, n_light = z["settings"]; v = z["camera"]
cam = Camera(position=v[0:3], look_at=v[3:6], up=v[6:9], fov_degrees=float(v[9]), width=int(v[10]), height=int(v[11]))
for mode in ("ours-aniso", "ours-iso"):
    st = RenderSettings(mode=mode, epsilon=float(eps), spp=int(spp), march_step=float(step), n_angular=int(n_ang),
                        seed=int(seed), n_inner=int(n_inner), n_light_samples=int(n_light), frozen=True)
    ref, rst = populate_cache(sc, cam, st)
    cs, pst = vdist.populate_sharded(sc, cam, st, window=3)
    ref3, st3 = populate_cache(sc, cam, st, window=3)
    for a, b in ((cs.single, ref.single), (cs.multiple, ref.multiple)):
        np.testing.assert_array_equal(a.packed(), b.packed())
    assert pst["records"] == rst["records"] > 0
    assert (pst["builds"], pst["windows"]) == (st3["builds"], st3["windows"])
dist.destroy_process_group()
print("populate sharded ok")
'''
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "populate sharded ok" in r.stdout
