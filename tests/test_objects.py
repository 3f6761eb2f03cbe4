"""ObjectRegistry on a device model (ref model.py:326-404) vs the reference.

The reference's own registry ran the sequence in
tests/golden/make_golden.py::objects_cases: refresh every row's local pose,
move object 1, refresh the local poses of a subset of edited rows, permute
the rows, move object 2.  Moved rows exact; poses within the float64/float32
tolerance of tests/test_gpu_dynamics.py (the device rotation algebra rounds
differently from numpy's matmul in the last bits).
"""

import numpy as np
import pytest

from conftest import load_cases
from gpu_util import require_gpu

pytestmark = pytest.mark.gpu
CASES = load_cases("objects_cases")
FIELDS = ("means", "log_scales", "quaternions", "logit_opacities", "sh_coeffs", "light_visibility", "object_ids")


@pytest.mark.parametrize("c", CASES, ids=lambda c: c["name"])
def test_gpu_object_registry_matches_reference(c):
    require_gpu()
    import torch
    from paper_2604_02851_b200.model import DeviceModel
    from paper_2604_02851_b200.objects import ObjectRegistry
    from paper_2604_02851_b200.pool import PermuteRecord, apply_mutation
    from paper_2604_02851_b200.geometry import quat_from_axis_angle
    dev = torch.device("cuda", 0)
    m = DeviceModel(*(torch.from_numpy(np.array(c.a(f"init_{k}"))).to(dev) for k in FIELDS), c["active"], c["degree"])
    reg = ObjectRegistry()
    reg.set_transform(1, quat_from_axis_angle([0, 1, 0], 0.3), [0.5, 0.0, -0.2])
    reg.set_transform(2, quat_from_axis_angle([1, 0.2, 0], -0.7), [0.0, 0.4, 0.1])
    close = dict(rtol=2e-7, atol=1e-7)
    reg.refresh_locals(m)
    np.testing.assert_allclose(reg.local_means.cpu().numpy(), c.a("lm0"), rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(reg.local_rotations.cpu().numpy(), c.a("lr0"), rtol=1e-12, atol=1e-12)
    rows1 = reg.apply_transform(m, 1, c.a("q1"), c.a("t1"))
    np.testing.assert_array_equal(rows1, c.a("rows1"))
    np.testing.assert_allclose(m.means.cpu().numpy(), c.a("means1"), **close)
    np.testing.assert_allclose(m.quaternions.cpu().numpy(), c.a("quats1"), rtol=0, atol=2e-7)
    m.means.copy_(torch.from_numpy(np.array(c.a("means_edit"))))
    reg.refresh_locals(m, c.a("sub"))
    np.testing.assert_allclose(reg.local_means.cpu().numpy(), c.a("lm2"), rtol=1e-9, atol=1e-9)
    np.testing.assert_allclose(reg.local_rotations.cpu().numpy(), c.a("lr2"), rtol=1e-9, atol=1e-9)
    rec = PermuteRecord(c.a("perm"), c["active"])
    apply_mutation(m, rec)
    reg.resize(rec)
    rows2 = reg.apply_transform(m, 2, c.a("q2"), c.a("t2"))
    np.testing.assert_array_equal(rows2, c.a("rows2"))
    np.testing.assert_allclose(m.means.cpu().numpy(), c.a("means3"), **close)
    np.testing.assert_allclose(m.quaternions.cpu().numpy(), c.a("quats3"), rtol=0, atol=2e-7)
    np.testing.assert_allclose(reg.local_means.cpu().numpy(), c.a("lm3"), rtol=1e-9, atol=1e-9)
    with pytest.raises(KeyError):
        reg.apply_transform(m, 9, [1, 0, 0, 0], [0, 0, 0])
