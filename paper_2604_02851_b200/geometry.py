"""Host-side camera and quaternion types of the reference API.

Mirrors the public surface of ref pkg/src/splatstream/geometry.py that the
hot-path entry points take as arguments: CameraIntrinsics (geometry.py:111),
Pose (geometry.py:146), OrthoCamera (geometry.py:252), look_at
(geometry.py:184) and the quaternion helpers.  Conventions are the
reference's: world +Y up; camera +X right, +Y down, +Z forward; quaternions
(w, x, y, z) rotate camera/local frames into the world; pixel (i, j) has its
centre at (i + 0.5, j + 0.5).  Objects of the reference's own classes are
accepted everywhere by duck typing.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


def quat_normalize(q):
    q = np.asarray(q, np.float64)
    return q / np.linalg.norm(q, axis=-1, keepdims=True)


def quat_multiply(a, b):
    """Hamilton product; R(a*b) = R(a) R(b)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    w1, x1, y1, z1 = np.moveaxis(a, -1, 0)
    w2, x2, y2, z2 = np.moveaxis(b, -1, 0)
    return np.stack([w1 * w2 - x1 * x2 - y1 * y2 - z1 * z2,
                     w1 * x2 + x1 * w2 + y1 * z2 - z1 * y2,
                     w1 * y2 - x1 * z2 + y1 * w2 + z1 * x2,
                     w1 * z2 + x1 * y2 - y1 * x2 + z1 * w2], -1)


def quat_conjugate(q):
    return np.asarray(q, np.float64) * np.array([1.0, -1.0, -1.0, -1.0])


def quat_from_axis_angle(axis, angle):
    ax = np.asarray(axis, np.float64)
    ax = ax / np.linalg.norm(ax)
    return np.concatenate([[math.cos(angle / 2)], math.sin(angle / 2) * ax])


def quat_to_rotmat(q):
    """(..., 3, 3) rotation; the quaternion is normalised first."""
    w, x, y, z = np.moveaxis(quat_normalize(q), -1, 0)
    r = np.stack([
        1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
        2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
        2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)], -1)
    return r.reshape(r.shape[:-1] + (3, 3))


def rotmat_to_quat(R):
    """Unit quaternion with w >= 0 for a proper rotation matrix."""
    R = np.asarray(R, np.float64)
    tr = R[0, 0] + R[1, 1] + R[2, 2]
    if tr > 0:
        s = 2.0 * math.sqrt(tr + 1.0)
        q = [0.25 * s, (R[2, 1] - R[1, 2]) / s, (R[0, 2] - R[2, 0]) / s, (R[1, 0] - R[0, 1]) / s]
    else:
        i = int(np.argmax(np.diag(R)))
        j, k = (i + 1) % 3, (i + 2) % 3
        s = 2.0 * math.sqrt(1.0 + R[i, i] - R[j, j] - R[k, k])
        v = [0.0, 0.0, 0.0]
        v[i] = 0.25 * s
        v[j] = (R[j, i] + R[i, j]) / s
        v[k] = (R[k, i] + R[i, k]) / s
        q = [(R[k, j] - R[j, k]) / s] + v
    q = np.asarray(q)
    return quat_normalize(-q if q[0] < 0 else q)


def quat_rotate(q, v):
    return (quat_to_rotmat(q) @ np.asarray(v, np.float64)[..., None])[..., 0]


@dataclass(frozen=True)
class CameraIntrinsics:
    """Pinhole camera; fx = fy = (H/2)/tan(fov_y/2), principal point at the centre."""

    width: int
    height: int
    fov_y: float
    near: float = 0.05
    far: float = 100.0

    def __post_init__(self):
        if not 0 < self.near < self.far:
            raise ValueError("require 0 < near < far")
        if not 0 < self.fov_y < math.pi:
            raise ValueError("require 0 < fov_y < pi")

    @property
    def fy(self) -> float:
        return (self.height / 2.0) / math.tan(self.fov_y / 2.0)

    @property
    def fx(self) -> float:
        return self.fy

    @property
    def cx(self) -> float:
        return self.width / 2.0

    @property
    def cy(self) -> float:
        return self.height / 2.0


@dataclass(frozen=True)
class Pose:
    """Camera position (world) and camera->world quaternion."""

    position: np.ndarray
    quaternion: np.ndarray

    def __post_init__(self):
        object.__setattr__(self, "position", np.asarray(self.position, np.float64))
        object.__setattr__(self, "quaternion", quat_normalize(self.quaternion))

    def rotation(self) -> np.ndarray:
        return quat_to_rotmat(self.quaternion)

    def forward(self) -> np.ndarray:
        return self.rotation()[:, 2]

    def world_to_camera(self, p):
        return (np.asarray(p, np.float64) - self.position) @ self.rotation()


def look_at(eye, target, up=(0.0, 1.0, 0.0)) -> Pose:
    """Pose at `eye` looking at `target` (+Z forward, +Y image-down)."""
    eye = np.asarray(eye, np.float64)
    fwd = np.asarray(target, np.float64) - eye
    n = np.linalg.norm(fwd)
    if n < 1e-12:
        raise ValueError("eye and target coincide")
    fwd = fwd / n
    right = np.cross(fwd, np.asarray(up, np.float64))
    if np.linalg.norm(right) < 1e-8:
        right = np.cross(fwd, np.array([0.0, 0.0, 1.0]))
    right = right / np.linalg.norm(right)
    down = np.cross(fwd, right)
    return Pose(eye, rotmat_to_quat(np.stack([right, down, fwd], axis=1)))


@dataclass(frozen=True)
class OrthoCamera:
    """Orthographic light camera: +Z projects; u spans [-half_width, half_width]."""

    pose: Pose
    half_width: float
    half_height: float
    width: int
    height: int
    far: float
