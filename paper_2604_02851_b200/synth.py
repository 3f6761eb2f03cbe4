"""Seeded synthetic workloads of SURVEY.md §8d ("random field").

n Gaussians in front of a camera ring: z ~ U(3,6) m; x, y uniform inside the
frustum (fov_y 1.2 rad) at that depth; pixel sigma ~ LogNormal(ln 2, 0.5),
log_scale = ln(sigma_px z / f) + N(0, 0.2^2) per axis; quaternion =
normalize(N(0,1)^4); logit opacity ~ U(-1,2); DC ~ U(-0.5,0.5); rest ~
U(-0.05,0.05); visibility ~ Bernoulli(0.7).  The ground-truth model perturbs
DC by U(-0.3,0.3) and means by N(0, 0.01^2).  Light (0.3,-1,0.2), I = 0.6,
flat ambient 0.35, background (0.05,0.05,0.08).  Views look from a 0.3 m
ring at z = 0 toward (0, 0, 4.5).
"""

from __future__ import annotations

import math

import numpy as np

from .geometry import CameraIntrinsics, look_at
from .model import GaussianModel
from .render import LightState, flat_ambient_sh

BACKGROUND = np.array([0.05, 0.05, 0.08])
FOV_Y = 1.2


def random_field(n: int, sh_degree: int = 3, width: int = 1920, height: int = 1080, seed: int = 0,
                 object_fraction: float = 0.0) -> GaussianModel:
    rng = np.random.default_rng(seed)
    f = (height / 2.0) / math.tan(FOV_Y / 2.0)
    z = rng.uniform(3.0, 6.0, n)
    hy = z * (height / 2.0) / f
    hx = hy * width / height
    x = rng.uniform(-1.0, 1.0, n) * hx
    y = rng.uniform(-1.0, 1.0, n) * hy
    sig = np.exp(rng.normal(math.log(2.0), 0.5, n))
    ls = np.log(sig * z / f)[:, None] + rng.normal(0.0, 0.2, (n, 3))
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    B = (sh_degree + 1) ** 2
    sh = np.empty((n, 3, B), np.float32)
    sh[:, :, 0] = rng.uniform(-0.5, 0.5, (n, 3))
    if B > 1:
        sh[:, :, 1:] = rng.uniform(-0.05, 0.05, (n, 3, B - 1))
    ids = np.zeros(n, np.int32)
    if object_fraction > 0:
        k = int(n * object_fraction)
        ids[rng.choice(n, k, replace=False)] = rng.integers(1, 4, k)
    return GaussianModel(
        means=np.stack([x, y, z], 1).astype(np.float32), log_scales=ls.astype(np.float32),
        quaternions=q.astype(np.float32), logit_opacities=rng.uniform(-1.0, 2.0, n).astype(np.float32),
        sh_coeffs=sh, light_visibility=(rng.random(n) < 0.7).astype(np.float32), object_ids=ids,
        active_count=n, sh_degree=sh_degree)


def target_model(model: GaussianModel, seed: int = 1) -> GaussianModel:
    rng = np.random.default_rng(seed)
    t = model.copy()
    t.sh_coeffs[:, :, 0] += rng.uniform(-0.3, 0.3, t.sh_coeffs[:, :, 0].shape).astype(np.float32)
    t.means += rng.normal(0.0, 0.01, t.means.shape).astype(np.float32)
    return t


def light() -> LightState:
    return LightState(direction=[0.3, -1.0, 0.2], intensity=[0.6, 0.6, 0.6],
                      ambient_sh=flat_ambient_sh([0.35, 0.35, 0.35]))


def ring_poses(k: int, radius: float = 0.3, target=(0.0, 0.0, 4.5)):
    return [look_at([radius * math.cos(2 * math.pi * i / k), radius * math.sin(2 * math.pi * i / k), 0.0], target)
            for i in range(k)]


def intrinsics(width=1920, height=1080) -> CameraIntrinsics:
    return CameraIntrinsics(width=width, height=height, fov_y=FOV_Y, near=0.05, far=100.0)
