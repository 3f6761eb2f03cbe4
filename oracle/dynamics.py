"""CPU restatement of the dynamic-scene row updates (test infrastructure only).

  light_visibility  ref pkg/src/splatstream/render.py:350-368 with
                    OrthoCamera.project geometry.py:267-271
  rigid transform   ref model.py:557-572 (ObjectRegistry.apply_transform)
  local poses       ref model.py:539-555 (ObjectRegistry.refresh_locals)
"""

from __future__ import annotations

import numpy as np

from .raster import quat_rotmat


def quat_mul(a, b):
    aw, ax, ay, az = np.moveaxis(np.asarray(a, np.float64), -1, 0)
    bw, bx, by, bz = np.moveaxis(np.asarray(b, np.float64), -1, 0)
    return np.stack([aw * bw - ax * bx - ay * by - az * bz,
                     aw * bx + ax * bw + ay * bz - az * by,
                     aw * by - ax * bz + ay * bw + az * bx,
                     aw * bz + ax * by - ay * bx + az * bw], -1)


def _unit(q):
    q = np.asarray(q, np.float64)
    return q / np.linalg.norm(q, axis=-1, keepdims=True)


def light_visibility(means, depth_map, cam_pos, cam_quat, half_w, half_h, width, height, bias=0.02):
    """Binary lit flag per row (f32)."""
    R = quat_rotmat(_unit(cam_quat))
    pc = (np.asarray(means, np.float64) - np.asarray(cam_pos, np.float64)) @ R
    u = (pc[:, 0] / half_w * 0.5 + 0.5) * width
    v = (pc[:, 1] / half_h * 0.5 + 0.5) * height
    z = pc[:, 2]
    px = np.floor(u).astype(np.int64)
    py = np.floor(v).astype(np.int64)
    inside = (px >= 0) & (px < width) & (py >= 0) & (py < height) & (z >= 0)
    out = np.ones(means.shape[0], np.float32)
    out[inside] = (z[inside] <= depth_map[py[inside], px[inside]] + bias).astype(np.float32)
    return out


def apply_transform(means, quats, rows, local_means, local_rots, q, t):
    """Rewrite rows of one object from local poses; in place on f32 arrays."""
    qn = _unit(q)
    R = quat_rotmat(qn)
    means[rows] = (local_means[rows] @ R.T + np.asarray(t, np.float64)).astype(np.float32)
    quats[rows] = _unit(quat_mul(qn[None, :], local_rots[rows])).astype(np.float32)


def refresh_locals(means, quats, rows, local_means, local_rots, q, t):
    qn = _unit(q)
    R = quat_rotmat(qn)
    local_means[rows] = (means[rows].astype(np.float64) - np.asarray(t, np.float64)) @ R
    conj = qn * np.array([1.0, -1.0, -1.0, -1.0])
    local_rots[rows] = _unit(quat_mul(conj[None, :], quats[rows].astype(np.float64)))
