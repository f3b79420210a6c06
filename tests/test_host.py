"""CPU-side checks of the boundary: the C-ABI library loads and exports every declared
symbol, host-side SeedSequence → PCG64 matches numpy, scene packing and configs."""

from __future__ import annotations

import re
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT

HEADER = ROOT / "include" / "volcache_b200.h"


def declared_symbols():
    txt = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*|int64_t)\s+(vc_\w+)\s*\(", txt, re.M)))


def test_library_exports_every_declared_symbol():
    from paper_1805_09258_b200 import _lib

    L = _lib.lib()
    syms = declared_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.EXPORTS)
    assert L.vc_version() == 1


@pytest.mark.parametrize("words", [[0, 401, 5], [7], [0], [2, 401, 18999], [3, 211, 0, 12345, 7],
                                   [4294967295, 1, 2, 3, 4, 5, 6, 7]])
def test_seedseq_pcg64_matches_numpy(words):
    from paper_1805_09258_b200 import _lib
    from paper_1805_09258_b200.records import pcg64_state

    w = np.array(words, dtype=np.uint32)
    out = np.zeros(4, np.uint64)
    _lib.check(_lib.lib().vc_seed_states(1, _lib.ptr(w), len(words), _lib.ptr(out)))
    ref, _ = pcg64_state(np.random.SeedSequence(words if len(words) > 1 else words[0]))
    np.testing.assert_array_equal(out, ref)


def test_seed_states_reject_bad_word_count():
    from paper_1805_09258_b200 import _lib

    out = np.zeros(4, np.uint64)
    w = np.zeros(20, np.uint32)
    with pytest.raises(ValueError):
        _lib.check(_lib.lib().vc_seed_states(1, _lib.ptr(w), 20, _lib.ptr(out)))


def test_configs_shapes():
    from paper_1805_09258_b200 import configs

    c1 = configs.cfg1()
    assert c1.points.shape == (256, 2) and c1.n_angular == 1024
    c2 = configs.cfg2()
    assert c2.points.shape == (4096, 3) and len(c2.scene.surfaces) == 14
    sc = configs.cfg3_scene()
    n_em = sum(1 for s in sc.surfaces if s.is_emitter)
    assert n_em == 16  # 8 windows × 2 triangles
    assert len(sc.surfaces) > 51200
    assert np.all(np.array([s.vertices for s in sc.surfaces]) >= -1e-12)


def test_scene_json_roundtrip(tmp_path):
    from paper_1805_09258_b200 import configs
    from paper_1805_09258_b200.scene import load_scene, save_scene, scene_arrays

    sc = configs.cfg2_scene()
    save_scene(sc, tmp_path / "s.json")
    back = load_scene(tmp_path / "s.json")
    for a, b in zip(scene_arrays(sc), scene_arrays(back)):
        np.testing.assert_array_equal(np.asarray(a), np.asarray(b))


def test_build_params_layout():
    import ctypes as C

    from paper_1805_09258_b200 import _lib

    # matches vc_build_params in include/volcache_b200.h (x86-64 SysV layout)
    assert C.sizeof(_lib.BuildParams) == 56  # include/volcache_b200.h vc_build_params (incl. media_bounces, hg_g)
    assert _lib.BuildParams.epsilon.offset == 24
    assert C.sizeof(_lib.Camera) == 10 * 8 + 6 * 4 + 4 * 0 or C.sizeof(_lib.Camera) == 104
