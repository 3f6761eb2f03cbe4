"""GSM1 model container (ref pkg/src/splatstream/model.py:407-442): save_model
bytes equal the unmodified reference's (tests/golden/make_gsm1.py) and
load_model round-trips them; host here, a DeviceModel on the GPU."""

import os

import numpy as np
import pytest

from gpu_util import require_gpu

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
NAMES = ("means", "log_scales", "quaternions", "logit_opacities", "sh_coeffs", "light_visibility", "object_ids")


def _case(deg):
    from paper_2604_02851_b200.model import GaussianModel
    z = np.load(os.path.join(HERE, "gsm1_cases.npz"))
    n, a, d = (int(x) for x in z[f"deg{deg}_meta"])
    return GaussianModel(*(z[f"deg{deg}_{k}"] for k in NAMES), a, d)


@pytest.mark.parametrize("deg", [1, 3])
def test_gsm1_save_matches_reference_bytes(deg, tmp_path):
    from paper_2604_02851_b200.model import load_model, save_model
    m = _case(deg)
    p = tmp_path / "m.gsm"
    save_model(p, m)
    ref = open(os.path.join(HERE, f"gsm1_deg{deg}.bin"), "rb").read()
    assert p.read_bytes() == ref
    back = load_model(os.path.join(HERE, f"gsm1_deg{deg}.bin"))
    assert (back.active_count, back.sh_degree, back.count) == (m.active_count, m.sh_degree, m.count)
    for k in NAMES:
        np.testing.assert_array_equal(getattr(back, k), getattr(m, k))
        assert getattr(back, k).dtype == getattr(m, k).dtype


def test_gsm1_rejects_other_containers(tmp_path):
    from paper_2604_02851_b200.model import load_model
    p = tmp_path / "x.bin"
    p.write_bytes(b"NOPE" + bytes(12))
    with pytest.raises(ValueError, match="not a model container"):
        load_model(p)


@pytest.mark.gpu
@pytest.mark.parametrize("deg", [1, 3])
def test_gpu_gsm1_device_round_trip(deg, tmp_path):
    require_gpu()
    from paper_2604_02851_b200.model import DeviceModel, load_model, save_model
    m = _case(deg)
    dm = load_model(os.path.join(HERE, f"gsm1_deg{deg}.bin"), device=0)
    assert isinstance(dm, DeviceModel)
    p = tmp_path / "d.gsm"
    save_model(p, dm)
    assert p.read_bytes() == open(os.path.join(HERE, f"gsm1_deg{deg}.bin"), "rb").read()
    for k in NAMES:
        np.testing.assert_array_equal(getattr(dm, k).cpu().numpy().reshape(getattr(m, k).shape), getattr(m, k))
