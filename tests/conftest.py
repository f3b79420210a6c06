"""Shared test setup: `gpu` marker, repo-root imports, golden fixture loader."""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libvolcache_b200.so")


def golden(name: str):
    return np.load(GOLDEN / f"{name}.npz", allow_pickle=False)


REC_CASES = ["cfg1_surf", "cfg1_m01", "pen2d", "refl2d", "cfg2_surf", "cfg2_m01",
             "cfg2_m01_canon", "box3d_refl", "room_small", "room_refl"]


def golden_scene(z, prefix=""):
    from paper_1805_09258_b200.scene import scene_from_arrays

    sig = z[prefix + "sigma"]
    lights = z[prefix + "lights"] if (prefix + "lights") in getattr(z, "files", z) else ()
    return scene_from_arrays(z[prefix + "verts"], z[prefix + "emission"], z[prefix + "albedo"],
                             z[prefix + "bmin"], z[prefix + "bmax"], sig[0], sig[1], lights)


def rel_l2(a, b, floor=1e-12):
    a = np.asarray(a, float)
    b = np.asarray(b, float)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), floor))


@pytest.fixture
def gold():
    return golden
