"""Scene descriptions for the ray-cast engine stand-in (ref scene.py).

The classes carry the fields the engine reads (ref scene.py:28-161 shapes
and albedo, 166-203 animation, 213-247 light and scene); the engine itself
only duck-types them, so the reference's own SceneDescription objects work
unchanged.  `scene_from_dict` reads the reference's YAML/dict layout
(ref scene.py:300-320).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from .geometry import quat_from_axis_angle, quat_to_rotmat


def _unit(v):
    v = np.asarray(v, dtype=np.float64)
    return v / np.linalg.norm(v)


def _arr(obj, name):
    object.__setattr__(obj, name, np.asarray(getattr(obj, name), dtype=np.float64))


@dataclass(frozen=True)
class Plane:
    """Infinite plane, or a rectangle of half sizes `extent` along tangents u, v."""

    point: np.ndarray
    normal: np.ndarray
    extent: Optional[tuple] = None

    def __post_init__(self):
        _arr(self, "point")
        object.__setattr__(self, "normal", _unit(self.normal))

    def tangents(self):
        """(u, v) as ref scene.py:41-46 (u = unit(ref x n), v = n x u)."""
        n = self.normal
        helper = np.array([1.0, 0, 0]) if abs(n[1]) > 0.9 else np.array([0, 1.0, 0])
        u = _unit(np.cross(helper, n))
        return u, np.cross(n, u)


@dataclass(frozen=True)
class Sphere:
    center: np.ndarray
    radius: float

    def __post_init__(self):
        _arr(self, "center")


@dataclass(frozen=True)
class Box:
    """Axis-aligned in the object's local frame."""

    center: np.ndarray
    half_extents: np.ndarray

    def __post_init__(self):
        _arr(self, "center")
        _arr(self, "half_extents")


@dataclass(frozen=True)
class Albedo:
    kind: str  # "solid" or "checker"
    color: np.ndarray = field(default_factory=lambda: np.array([0.7, 0.7, 0.7]))
    color2: np.ndarray = field(default_factory=lambda: np.array([0.2, 0.2, 0.2]))
    scale: float = 1.0

    def __post_init__(self):
        _arr(self, "color")
        _arr(self, "color2")


@dataclass(frozen=True)
class Animation:
    """Rigid motion script: none | rotate | bounce | oscillate (ref scene.py:166-203)."""

    kind: str = "none"
    axis: np.ndarray = field(default_factory=lambda: np.array([0.0, 1.0, 0.0]))
    anchor: np.ndarray = field(default_factory=lambda: np.zeros(3))
    deg_per_s: float = 0.0
    height: float = 0.0
    amplitude: float = 0.0
    period: float = 1.0

    def __post_init__(self):
        _arr(self, "axis")
        _arr(self, "anchor")

    def transform_at(self, time: float):
        """(quaternion wxyz, translation) local -> world at `time` seconds."""
        ident = np.array([1.0, 0, 0, 0])
        if self.kind == "none":
            return ident, np.zeros(3)
        if self.kind == "rotate":
            q = quat_from_axis_angle(self.axis, np.deg2rad(self.deg_per_s) * time)
            return q, self.anchor - quat_to_rotmat(q) @ self.anchor
        if self.kind == "bounce":
            return ident, np.array([0.0, self.height * abs(np.sin(np.pi * time / self.period)), 0.0])
        if self.kind == "oscillate":
            return ident, _unit(self.axis) * (self.amplitude * np.sin(2 * np.pi * time / self.period))
        raise ValueError(f"unknown animation kind {self.kind!r}")


@dataclass(frozen=True)
class SceneObject:
    object_id: int
    shape: object
    albedo: Albedo
    animation: Animation = field(default_factory=Animation)


@dataclass(frozen=True)
class DirectionalLight:
    direction: np.ndarray
    intensity: np.ndarray
    ambient: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "direction", _unit(self.direction))
        _arr(self, "intensity")
        _arr(self, "ambient")


@dataclass(frozen=True)
class SceneDescription:
    objects: tuple
    light: DirectionalLight
    background: np.ndarray = field(default_factory=lambda: np.zeros(3))

    def __post_init__(self):
        _arr(self, "background")
        ids = [o.object_id for o in self.objects if o.object_id > 0]
        if len(ids) != len(set(ids)):
            raise ValueError("dynamic object_ids must be unique")

    def dynamic_ids(self):
        return sorted(o.object_id for o in self.objects if o.object_id > 0)

    def transforms_at(self, time: float):
        return {o.object_id: o.animation.transform_at(time) for o in self.objects if o.object_id > 0}


def _shape(d):
    k = d["kind"]
    if k == "plane":
        return Plane(d["point"], d["normal"], tuple(d["extent"]) if d.get("extent") is not None else None)
    if k == "sphere":
        return Sphere(d["center"], float(d["radius"]))
    if k == "box":
        return Box(d["center"], d["half_extents"])
    raise ValueError(f"unknown shape kind {k!r}")


def _albedo(d):
    if d["kind"] == "solid":
        return Albedo("solid", color=d["color"])
    return Albedo("checker", color=d["colors"][0], color2=d["colors"][1], scale=float(d.get("scale", 1.0)))


def scene_from_dict(d: dict) -> SceneDescription:
    objs = tuple(SceneObject(int(o.get("id", 0)), _shape(o["shape"]), _albedo(o["albedo"]),
                             Animation(**o["animation"]) if o.get("animation") else Animation())
                 for o in d["objects"])
    ld = d["light"]
    return SceneDescription(objs, DirectionalLight(ld["direction"], ld["intensity"], ld["ambient"]),
                            np.asarray(d.get("background", [0, 0, 0]), dtype=np.float64))


def load_scene(path) -> SceneDescription:
    import yaml
    with open(path) as f:
        return scene_from_dict(yaml.safe_load(f))


__all__ = ["Plane", "Sphere", "Box", "Albedo", "Animation", "SceneObject", "DirectionalLight", "SceneDescription",
           "scene_from_dict", "load_scene"]
