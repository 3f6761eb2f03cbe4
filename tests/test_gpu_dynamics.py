"""GPU dynamics kernels vs the reference (golden) -- light visibility bit-exact,
rigid transforms within one float32 ulp."""

import numpy as np
import pytest

from conftest import load_cases
from gpu_util import require_gpu

pytestmark = pytest.mark.gpu
DYN = load_cases("dyn_cases")


@pytest.mark.parametrize("c", DYN, ids=[f"{c['kind']}_{c['n']}" for c in DYN])
def test_gpu_dynamics(c):
    require_gpu()
    import torch
    from paper_2604_02851_b200 import _lib
    from paper_2604_02851_b200.geometry import OrthoCamera, Pose
    from paper_2604_02851_b200.model import GaussianModel, DeviceModel
    from paper_2604_02851_b200.render import update_light_visibility
    n = c["n"]
    if c["kind"] == "lightvis":
        m = GaussianModel(c.a("means").copy(), np.zeros((n, 3), np.float32), np.tile(np.float32([1, 0, 0, 0]), (n, 1)),
                          np.zeros(n, np.float32), np.zeros((n, 3, 1), np.float32), np.zeros(n, np.float32),
                          np.zeros(n, np.int32), n, 0)
        cam = OrthoCamera(Pose(c.a("cam_pos"), c.a("cam_quat")), c["half_width"], c["half_height"], c["width"],
                          c["height"], 20.0)
        update_light_visibility(m, c.a("depth"), cam, c["bias"])
        np.testing.assert_array_equal(m.light_visibility, c.a("vis"))
    else:
        m = GaussianModel(c.a("means").copy(), np.zeros((n, 3), np.float32), c.a("quats").copy(),
                          np.zeros(n, np.float32), np.zeros((n, 3, 1), np.float32), np.ones(n, np.float32),
                          c.a("object_ids").copy(), n, 0)
        dm = DeviceModel.from_host(m)
        lm = torch.from_numpy(c.a("local_means")).cuda()
        lr = torch.from_numpy(c.a("local_rots")).cuda()
        ctx = _lib.ctx()
        q = (_lib.f64 * 4)(*c.a("q"))
        t = (_lib.f64 * 3)(*c.a("t"))
        ctx.check(ctx.lib.ss_apply_object_transform(ctx.handle, dm.struct(), c["oid"], _lib.ptr(lm), _lib.ptr(lr), q, t))
        out = dm.to_host()
        np.testing.assert_allclose(out.means, c.a("out_means"), rtol=2e-7, atol=1e-7)
        np.testing.assert_allclose(out.quaternions, c.a("out_quats"), rtol=0, atol=2e-7)


def test_gpu_light_visibility_change_flag():
    """ref server.py:406-409 on the device: the flag is set exactly when a
    visibility bit flips (against the values before the update)."""
    require_gpu()
    import torch
    from paper_2604_02851_b200.geometry import OrthoCamera, Pose
    from paper_2604_02851_b200.model import DeviceModel, GaussianModel
    from paper_2604_02851_b200.render import update_light_visibility
    c = [x for x in DYN if x["kind"] == "lightvis" and x["n"] == 1000][0]
    n = c["n"]
    m = GaussianModel(c.a("means").copy(), np.zeros((n, 3), np.float32), np.tile(np.float32([1, 0, 0, 0]), (n, 1)),
                      np.zeros(n, np.float32), np.zeros((n, 3, 1), np.float32), np.zeros(n, np.float32),
                      np.zeros(n, np.int32), n, 0)
    dm = DeviceModel.from_host(m)
    cam = OrthoCamera(Pose(c.a("cam_pos"), c.a("cam_quat")), c["half_width"], c["half_height"], c["width"],
                      c["height"], 20.0)
    depth = torch.from_numpy(np.array(c.a("depth"))).cuda()
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    update_light_visibility(dm, depth, cam, c["bias"], changed=flag)  # from all-zero: bits flip
    assert int(flag.item()) == 1
    np.testing.assert_array_equal(dm.light_visibility.cpu().numpy(), c.a("vis"))
    flag.zero_()
    update_light_visibility(dm, depth, cam, c["bias"], changed=flag)  # same light: no change
    assert int(flag.item()) == 0
    dm.light_visibility[n // 2] = 1.0 - dm.light_visibility[n // 2]  # one row differs from what the map gives
    update_light_visibility(dm, depth, cam, c["bias"], changed=flag)
    assert int(flag.item()) == 1
