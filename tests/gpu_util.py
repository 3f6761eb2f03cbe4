"""Helpers for the -m gpu parity tests (build product arguments from golden cases)."""

import numpy as np

from conftest import NS, case_model
from oracle import raster as orr


def require_gpu():
    import pytest
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2604_02851_b200 import _lib
    _lib.load_library()  # raises if the library is missing: no silent fallback


def product_args(c):
    from paper_2604_02851_b200.geometry import CameraIntrinsics, Pose
    from paper_2604_02851_b200.model import GaussianModel
    from paper_2604_02851_b200.render import LightState
    m = case_model(c)
    model = GaussianModel(m.means, m.log_scales, m.quaternions, m.logit_opacities, m.sh_coeffs,
                          m.light_visibility, m.object_ids, m.active_count, m.sh_degree)
    p = c.a("pose")
    pose = Pose(p[:3], p[3:])
    intr = CameraIntrinsics(width=c["W"], height=c["H"], fov_y=c["fov"], near=c["near"])
    light = LightState(c.a("light_dir"), c.a("light_int"), c.a("ambient") if c.has("ambient") else None)
    # golden directions are already unit vectors; keep the exact doubles
    light.direction = np.array(c.a("light_dir"), np.float64)
    return model, pose, intr, light


def oracle_args(c, pose, intr):
    cam = orr.camera(pose, intr)
    light = dict(direction=c.a("light_dir"), intensity=c.a("light_int"),
                 ambient=c.a("ambient") if c.has("ambient") else None)
    return case_model(c), cam, light
