"""Host-side scene model mirroring the reference's `volcache.scene` types.

Only what the GPU path needs: surfaces (segments in 2D, triangles in 3D) with
RGB emission/albedo, a homogeneous medium and an axis-aligned bounds box.
The classes are duck-compatible with the reference (`src/scene.py:41-219`), so a
reference `Scene` object can be passed to every entry point of this package
unchanged, and scene JSON files use the reference format (`src/scene.py:441-536`).
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

LUMINANCE_WEIGHTS = np.array([0.2126, 0.7152, 0.0722])  # src/scene.py:24


class SceneFormatError(ValueError):
    """Malformed scene description (src/scene.py:27-28)."""


def _rgb(v, name):
    a = np.asarray(v, dtype=float)
    if a.ndim == 0:
        a = np.full(3, float(a))
    if a.shape != (3,):
        raise SceneFormatError(f"{name} must be a scalar or a 3-vector")
    return a


@dataclass(frozen=True)
class Medium:
    sigma_s: float
    sigma_a: float

    def __post_init__(self):
        if self.sigma_s < 0.0 or self.sigma_a < 0.0:
            raise ValueError("medium coefficients must be non-negative")

    @property
    def sigma_t(self) -> float:
        return self.sigma_s + self.sigma_a


@dataclass(frozen=True)
class Surface:
    vertices: np.ndarray
    emission: np.ndarray = field(default_factory=lambda: np.zeros(3))
    albedo: np.ndarray = field(default_factory=lambda: np.zeros(3))

    def __post_init__(self):
        v = np.asarray(self.vertices, dtype=float)
        if v.shape not in ((2, 2), (3, 3)):
            raise SceneFormatError("vertices must be a 2D segment or a 3D triangle")
        object.__setattr__(self, "vertices", v)
        object.__setattr__(self, "emission", _rgb(self.emission, "emission"))
        object.__setattr__(self, "albedo", _rgb(self.albedo, "albedo"))
        if np.any(self.emission < 0.0):
            raise SceneFormatError("emission must be non-negative")
        if np.any(self.albedo < 0.0) or np.any(self.albedo > 1.0):
            raise SceneFormatError("albedo must lie in [0, 1]")

    @property
    def dim(self) -> int:
        return self.vertices.shape[1]

    @property
    def is_emitter(self) -> bool:
        return bool(np.any(self.emission > 0.0))


@dataclass
class Scene:
    surfaces: tuple
    medium: Medium
    bounds_min: np.ndarray
    bounds_max: np.ndarray
    # extension (the reference has area emitters only): delta lights as rows
    # (kind, v0, v1, v2, r, g, b, 0) — see point_light / directional_light
    lights: np.ndarray = field(default_factory=lambda: np.zeros((0, 8)))

    def __post_init__(self):
        self.surfaces = tuple(self.surfaces)
        self.lights = np.asarray(self.lights, dtype=float).reshape(-1, 8)
        self.bounds_min = np.asarray(self.bounds_min, dtype=float)
        self.bounds_max = np.asarray(self.bounds_max, dtype=float)
        if self.bounds_min.shape != self.bounds_max.shape or self.bounds_min.ndim != 1:
            raise SceneFormatError("bounds min/max must be vectors of equal length")
        if self.bounds_min.size not in (2, 3):
            raise SceneFormatError("dimensionality must be 2 or 3")
        if np.any(self.bounds_max <= self.bounds_min):
            raise SceneFormatError("bounds max must exceed min on every axis")

    @property
    def dim(self) -> int:
        return self.bounds_min.size

    @property
    def scale(self) -> float:
        return float(np.linalg.norm(self.bounds_max - self.bounds_min))

    @property
    def max_emission(self) -> float:
        return float(max((np.max(s.emission) for s in self.surfaces), default=0.0))

    def contains(self, points) -> np.ndarray:
        pts = np.atleast_2d(np.asarray(points, dtype=float))
        eps = 1e-12 * self.scale
        ok = np.all((pts >= self.bounds_min - eps) & (pts <= self.bounds_max + eps), axis=1)
        return ok if np.asarray(points).ndim == 2 else bool(ok[0])


def point_light(position, intensity) -> np.ndarray:
    """Extension: an isotropic point light (radiant intensity rgb) as a Scene.lights row."""
    p = np.zeros(3)
    v = np.asarray(position, float)
    p[: v.size] = v
    return np.concatenate([[0.0], p, _rgb(intensity, "intensity"), [0.0]])


def directional_light(toward, irradiance) -> np.ndarray:
    """Extension: a distant light; `toward` points from the scene to the light (normalised
    here), `irradiance` is the rgb irradiance on a plane facing it."""
    v = np.asarray(toward, float)
    v = v / np.linalg.norm(v)
    p = np.zeros(3)
    p[: v.size] = v
    return np.concatenate([[1.0], p, _rgb(irradiance, "irradiance"), [0.0]])


def scene_arrays(scene):
    """Packed float64 arrays of any duck-typed scene: verts (K,k,d), emission, albedo."""
    dim = int(np.asarray(scene.bounds_min).size)
    surfs = list(scene.surfaces)
    if not surfs:
        return dim, np.zeros((0, dim, dim)), np.zeros((0, 3)), np.zeros((0, 3))
    verts = np.ascontiguousarray(
        np.array([np.asarray(s.vertices, float) for s in surfs]).reshape(-1, dim, dim)
    )
    em = np.ascontiguousarray(np.array([_rgb(s.emission, "emission") for s in surfs]))
    al = np.ascontiguousarray(np.array([_rgb(s.albedo, "albedo") for s in surfs]))
    return dim, verts, em, al


def scene_from_arrays(verts, emission, albedo, bounds_min, bounds_max, sigma_s, sigma_a, lights=()) -> Scene:
    return Scene(
        lights=np.asarray(lights, float).reshape(-1, 8),
        surfaces=tuple(
            Surface(vertices=v, emission=e, albedo=a) for v, e, a in zip(verts, emission, albedo)
        ),
        medium=Medium(float(sigma_s), float(sigma_a)),
        bounds_min=np.asarray(bounds_min, float),
        bounds_max=np.asarray(bounds_max, float),
    )


def scene_to_dict(scene) -> dict:
    d = _scene_to_dict(scene)
    lights = getattr(scene, "lights", None)
    if lights is not None and len(lights):  # extension key, absent for reference scenes
        d["lights"] = np.asarray(lights, float).reshape(-1, 8).tolist()
    return d


def _scene_to_dict(scene) -> dict:
    return {
        "dimensionality": int(np.asarray(scene.bounds_min).size),
        "medium": {"sigma_s": float(scene.medium.sigma_s), "sigma_a": float(scene.medium.sigma_a)},
        "bounds": {
            "min": np.asarray(scene.bounds_min, float).tolist(),
            "max": np.asarray(scene.bounds_max, float).tolist(),
        },
        "surfaces": [
            {
                "vertices": np.asarray(s.vertices, float).tolist(),
                "emission": _rgb(s.emission, "emission").tolist(),
                "albedo": _rgb(s.albedo, "albedo").tolist(),
            }
            for s in scene.surfaces
        ],
    }


def scene_from_dict(d: dict) -> Scene:
    try:
        dim = d["dimensionality"]
        med = d["medium"]
        b = d["bounds"]
        raw = d["surfaces"]
    except (KeyError, TypeError) as exc:
        raise SceneFormatError(f"malformed scene: {exc}") from exc
    if dim not in (2, 3):
        raise SceneFormatError("dimensionality must be 2 or 3")
    surfs = []
    for i, s in enumerate(raw):
        v = np.asarray(s["vertices"], float)
        if v.ndim != 2 or v.shape[1] != dim:
            raise SceneFormatError(f"surface {i} vertices must be points of dim {dim}")
        surfs.append(Surface(vertices=v, emission=s.get("emission", 0.0), albedo=s.get("albedo", 0.0)))
    return Scene(
        surfaces=tuple(surfs),
        medium=Medium(float(med.get("sigma_s", 0.0)), float(med.get("sigma_a", 0.0))),
        bounds_min=np.asarray(b["min"], float),
        bounds_max=np.asarray(b["max"], float),
        lights=np.asarray(d.get("lights", []), float).reshape(-1, 8),
    )


def load_scene(path) -> Scene:
    return scene_from_dict(json.loads(Path(path).read_text()))


def save_scene(scene, path) -> None:
    Path(path).write_text(json.dumps(scene_to_dict(scene), indent=1) + "\n")
