"""Cache persistence and image I/O (src/cache.py:397-491, src/renderer.py:689-730), CPU-only.

Mirrors the reference's serialization and PFM tests (tests/test_cache.py:663-760,
tests/test_renderer.py:513-560) and reads files written by the reference itself
(tests/golden/ref_cache.json, ref_image.pfm; make_goldens.py gen_io).
"""

from __future__ import annotations

import json

import numpy as np
import pytest

from conftest import GOLDEN
from paper_1805_09258_b200.cache import RadianceCache
from paper_1805_09258_b200.io import (CACHE_FORMAT, CACHE_VERSION, BaselineRecord, CacheFormatError, load_cache,
                                      load_cache_npz, read_pfm, save_cache, save_cache_npz, write_pfm, write_ppm)
from paper_1805_09258_b200.records import CacheRecord


def _ellipse(position=(0.5, 0.5), angle=0.4, radii=(0.2, 0.1)):
    c, s = np.cos(angle), np.sin(angle)
    return CacheRecord(position=np.array(position, float), value=np.array([1.0, 0.5, 0.25]),
                       grad=np.arange(6.0).reshape(3, 2) / 7.0, axes=np.array([[c, -s], [s, c]]),
                       radii=np.array(radii, float))


def test_cache_round_trip(tmp_path):
    cache = RadianceCache(np.array([0.0, -1.0]), np.array([2.0, 3.0]))
    cache.insert(_ellipse())
    cache.insert(BaselineRecord(position=np.array([1.0, 2.0]), value=np.array([0.5, 0.25, 0.125]),
                                grad=np.ones((3, 2)), radius=0.15))
    path = tmp_path / "cache.json"
    save_cache(cache, path, metadata={"mode": "test", "epsilon": 0.01})
    loaded, meta = load_cache(path)
    assert meta == {"mode": "test", "epsilon": 0.01}
    assert loaded.dim == 2 and len(loaded) == 2
    np.testing.assert_array_equal(loaded.bounds_min, cache.bounds_min)
    e0, s0 = cache.records
    e1, s1 = loaded.records
    assert isinstance(e1, CacheRecord) and isinstance(s1, BaselineRecord)
    for f in ("position", "value", "grad", "axes", "radii"):
        np.testing.assert_array_equal(getattr(e1, f), getattr(e0, f))
    assert s1.radius == s0.radius
    np.testing.assert_array_equal(loaded.packed(), cache.packed())


def test_reads_reference_written_cache(tmp_path):
    loaded, meta = load_cache(GOLDEN / "ref_cache.json")
    assert meta == {"mode": "test", "epsilon": 0.01}
    e, s = loaded.records
    np.testing.assert_array_equal(e.radii, [0.2, 0.1])
    assert isinstance(s, BaselineRecord) and s.radius == 0.15
    # re-saving gives the reference's document back, byte for byte
    out = tmp_path / "again.json"
    save_cache(loaded, out, metadata=meta)
    assert out.read_text() == (GOLDEN / "ref_cache.json").read_text()


def test_save_cache_default_metadata(tmp_path):
    cache = RadianceCache(np.zeros(2), np.ones(2))
    path = tmp_path / "empty.json"
    save_cache(cache, path)
    loaded, meta = load_cache(path)
    assert meta == {} and len(loaded) == 0
    doc = json.loads(path.read_text())
    assert doc["format"] == CACHE_FORMAT and doc["version"] == CACHE_VERSION


def test_load_cache_rejects_bad_documents(tmp_path):
    def write(name, payload):
        p = tmp_path / name
        p.write_text(payload if isinstance(payload, str) else json.dumps(payload))
        return p

    with pytest.raises(CacheFormatError):
        load_cache(write("notjson.json", "{this is not json"))
    with pytest.raises(CacheFormatError):
        load_cache(write("list.json", [1, 2, 3]))
    with pytest.raises(CacheFormatError):
        load_cache(write("fmt.json", {"format": "something-else", "version": 1}))
    good = {"format": CACHE_FORMAT, "version": CACHE_VERSION, "dimensionality": 2,
            "bounds": {"min": [0.0, 0.0], "max": [1.0, 1.0]}, "metadata": {}, "records": []}
    with pytest.raises(CacheFormatError):
        load_cache(write("future.json", dict(good, version=CACHE_VERSION + 1)))
    with pytest.raises(CacheFormatError):
        load_cache(write("dims.json", dict(good, dimensionality=3)))
    with pytest.raises(CacheFormatError):
        load_cache(write("nobounds.json", {k: v for k, v in good.items() if k != "bounds"}))
    with pytest.raises(OSError):
        load_cache(tmp_path / "does-not-exist.json")


def test_load_cache_rejects_bad_records(tmp_path):
    ok = {"record_type": "ellipsoid", "position": [0.5, 0.5], "value": [1.0, 1.0, 1.0],
          "grad": [[0.0, 0.0]] * 3, "axes": [[1.0, 0.0], [0.0, 1.0]], "radii": [0.1, 0.1]}

    def doc_with(record):
        return {"format": CACHE_FORMAT, "version": CACHE_VERSION, "dimensionality": 2,
                "bounds": {"min": [0.0, 0.0], "max": [1.0, 1.0]}, "metadata": {}, "records": [record]}

    for name, mutate in [("nopos", lambda d: d.pop("position")), ("shortpos", lambda d: d.update(position=[0.5])),
                         ("shortval", lambda d: d.update(value=[1.0])),
                         ("shortgrad", lambda d: d.update(grad=[[0.0, 0.0]])),
                         ("shortradii", lambda d: d.update(radii=[0.1])),
                         ("badtype", lambda d: d.update(record_type="cylinder"))]:
        bad = json.loads(json.dumps(ok))
        mutate(bad)
        p = tmp_path / f"{name}.json"
        p.write_text(json.dumps(doc_with(bad)))
        with pytest.raises(CacheFormatError):
            load_cache(p)
    p = tmp_path / "good.json"
    p.write_text(json.dumps(doc_with(ok)))
    loaded, _ = load_cache(p)
    assert len(loaded) == 1


def test_npz_sidecar_round_trip(tmp_path):
    cache = RadianceCache(np.zeros(3), np.ones(3))
    rng = np.random.default_rng(3)
    for _ in range(5):
        q, _ = np.linalg.qr(rng.normal(size=(3, 3)))
        cache.insert(CacheRecord(rng.uniform(0, 1, 3), rng.uniform(0, 1, 3), rng.normal(size=(3, 3)), q,
                                 rng.uniform(0.05, 0.3, 3)))
    p = tmp_path / "c.npz"
    save_cache_npz(cache, p, tags=np.arange(5))
    back = load_cache_npz(p)
    np.testing.assert_array_equal(back.packed(), cache.packed())
    assert np.load(p)["tags"].tolist() == [0, 1, 2, 3, 4]


def test_pfm_round_trip_and_reference_file(tmp_path):
    ref = read_pfm(GOLDEN / "ref_image.pfm")
    img = np.random.default_rng(0).uniform(0.0, 10.0, size=(5, 7, 3)).astype(np.float32)
    np.testing.assert_array_equal(ref, img)
    p = tmp_path / "img.pfm"
    write_pfm(p, img)
    assert p.read_bytes() == (GOLDEN / "ref_image.pfm").read_bytes()
    back = read_pfm(p)
    assert back.dtype == np.float32 and np.array_equal(back, img)


def test_pfm_header_and_bad_input(tmp_path):
    p = tmp_path / "img.pfm"
    write_pfm(p, np.zeros((2, 3, 3), np.float32))
    raw = p.read_bytes()
    assert raw.startswith(b"PF\n3 2\n-1.0\n") and len(raw) == len(b"PF\n3 2\n-1.0\n") + 72
    with pytest.raises(ValueError):
        write_pfm(tmp_path / "x.pfm", np.zeros((4, 4)))
    bad = tmp_path / "bad.pfm"
    bad.write_bytes(b"Pf\n1 1\n-1.0\n" + b"\x00" * 4)
    with pytest.raises(ValueError):
        read_pfm(bad)
    tr = tmp_path / "trunc.pfm"
    tr.write_bytes(b"PF\n2 2\n-1.0\n" + b"\x00" * 8)
    with pytest.raises(ValueError):
        read_pfm(tr)


def test_write_ppm(tmp_path):
    image = np.zeros((2, 2, 3))
    image[0, 0] = 1.0
    p = tmp_path / "img.ppm"
    write_ppm(p, image)
    raw = p.read_bytes()
    assert raw.startswith(b"P6\n2 2\n255\n")
    payload = raw[len(b"P6\n2 2\n255\n"):]
    assert payload[:3] == b"\xff\xff\xff" and payload[3:6] == b"\x00\x00\x00"
    with pytest.raises(ValueError):
        write_ppm(tmp_path / "y.ppm", np.zeros((2, 2)))


def test_render_settings_and_targets_validation():
    from paper_1805_09258_b200.renderer import Camera, CacheSet, FieldGrid, RenderSettings

    with pytest.raises(ValueError):
        RenderSettings(mode="nope")
    with pytest.raises(ValueError):
        RenderSettings(epsilon=0.0)
    with pytest.raises(ValueError):
        RenderSettings(march_step=-1.0)
    with pytest.raises(ValueError):
        RenderSettings(spp=0)
    with pytest.raises(ValueError):
        FieldGrid(np.zeros(3), np.ones(3), 2, 2)
    with pytest.raises(ValueError):
        FieldGrid(np.zeros(2), np.zeros(2), 2, 2)
    with pytest.raises(ValueError):
        FieldGrid(np.zeros(2), np.ones(2), 0, 2)
    g = FieldGrid(np.zeros(2), np.ones(2), 4, 2)
    np.testing.assert_allclose(g.cell_center(0, 0), [0.125, 0.75])
    np.testing.assert_array_equal(g.centers[1, 3], g.cell_center(1, 3))
    for kw in (dict(fov_degrees=0.0), dict(fov_degrees=180.0), dict(width=0), dict(look_at=np.array([0.5, 0.5, 0.5])),
               dict(up=np.array([0.0, 0.0, 1.0])), dict(position=np.zeros(2))):
        base = dict(position=np.array([0.5, 0.5, 0.5]), look_at=np.array([0.5, 0.5, 1.0]),
                    up=np.array([0.0, 1.0, 0.0]), fov_degrees=60.0, width=2, height=2)
        base.update(kw)
        with pytest.raises(ValueError):
            Camera(**base)
    with pytest.raises(ValueError):
        CacheSet(None, "path")
