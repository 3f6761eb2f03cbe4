"""Pool maintenance on a device model vs the reference.

Expectations are the unmodified reference's own outcomes
(tests/golden/make_golden.py::pool_cases): GridIndex.rebuild's cell map,
precull (with and without engine depth buffers), freeze_policy, freeze_range
(+ OptimizerState.resize, DeltaBaselines.apply_record), prune, a client-side
placeholder append, and the ordering packet bytes.  Exact equality.
"""

import numpy as np
import pytest

from conftest import load_cases
from gpu_util import require_gpu

pytestmark = pytest.mark.gpu

CASES = load_cases("pool_cases")
FIELDS = ("means", "log_scales", "quaternions", "logit_opacities", "sh_coeffs", "light_visibility", "object_ids")
GROUPS = ("means", "log_scales", "quaternions", "logit_opacities", "sh_coeffs")


def _model(c, prefix=""):
    import torch
    from paper_2604_02851_b200.model import DeviceModel
    t = lambda k: torch.from_numpy(np.array(c.a(prefix + k))).to(torch.device("cuda", 0))
    return DeviceModel(*(t(k) for k in FIELDS), c["active"], c["degree"])


def _opt(c, m, prefix="opt_"):
    import torch
    from paper_2604_02851_b200.optim import OptimizerState
    o = OptimizerState(m, scene_extent=3.0)
    for k in GROUPS:  # the reference-visible numpy state, written back on the next device use
        o.m[k][...] = c.a(f"{prefix}m_{k}")
        o.v[k][...] = c.a(f"{prefix}v_{k}")
    o.age[...] = c.a(f"{prefix}age")
    o.grad_ema[...] = c.a(f"{prefix}grad_ema")
    return o


def _check_model(m, c, prefix, active):
    assert m.active_count == active
    for k in FIELDS:
        np.testing.assert_array_equal(getattr(m, k).cpu().numpy(), c.a(prefix + k), err_msg=prefix + k)


def _check_opt(o, c, prefix):
    for k in GROUPS:
        np.testing.assert_array_equal(o.m[k], c.a(f"{prefix}m_{k}"), err_msg=k)
        np.testing.assert_array_equal(o.v[k], c.a(f"{prefix}v_{k}"), err_msg=k)
    np.testing.assert_array_equal(o.age, c.a(f"{prefix}age"))
    np.testing.assert_array_equal(o.grad_ema, c.a(f"{prefix}grad_ema"))


def _baselines(c):
    import torch
    from paper_2604_02851_b200.protocol import DeviceBaselines
    dev = torch.device("cuda", 0)
    return DeviceBaselines(torch.from_numpy(np.array(c.a("base_means"))).to(dev),
                           torch.from_numpy(np.array(c.a("base_log_scales"))).to(dev), 1)


@pytest.mark.parametrize("c", CASES, ids=lambda c: c["name"])
def test_gpu_grid_and_precull(c):
    require_gpu()
    from paper_2604_02851_b200 import pool
    from paper_2604_02851_b200.geometry import CameraIntrinsics, Pose
    m = _model(c)
    g = pool.GridIndex(cell_size=c["cell"], origin=c["origin"])
    g.rebuild(m)
    keys, lens, rows = c.a("cell_keys"), c.a("cell_lens"), c.a("cell_rows")
    cm = g.cell_map
    assert list(cm.keys()) == [tuple(int(v) for v in k) for k in keys.reshape(-1, 3)]  # dict order too
    assert [len(v) for v in cm.values()] == lens.tolist()
    got_rows = np.concatenate([np.array(v, np.int64) for v in cm.values()]) if cm else np.zeros(0, np.int64)
    np.testing.assert_array_equal(got_rows, rows)
    intr = CameraIntrinsics(width=c["width"], height=c["height"], fov_y=c["fov_y"], near=c["near"], far=c["far"])
    poses = [Pose(p[:3], p[3:]) for p in c.a("poses")]
    np.testing.assert_array_equal(pool.precull(m, g, poses, intr), c.a("precull"))
    np.testing.assert_array_equal(pool.precull(m, g, poses, intr, as_tensor=True).cpu().numpy(), c.a("precull"))
    np.testing.assert_array_equal(pool.precull(m, g, poses, intr, [c.a("depth0"), c.a("depth1")]),
                                  c.a("precull_depth"))


@pytest.mark.parametrize("c", CASES, ids=lambda c: c["name"])
def test_gpu_freeze_and_resize(c):
    require_gpu()
    from paper_2604_02851_b200 import pool
    m = _model(c)
    o = _opt(c, m)
    b = _baselines(c)
    frz = pool.freeze_policy(m, o, age_threshold=120, grad_threshold=3e-4)
    np.testing.assert_array_equal(frz, c.a("freeze"))
    rec = pool.freeze_range(m, frz)
    assert (rec is not None) == c["has_permute"]
    if rec is not None:
        np.testing.assert_array_equal(rec.permutation, c.a("permutation"))
        o.resize(rec)
        pool.baselines_apply_record(b, rec)
    _check_model(m, c, "frozen_", c["frozen_active"])
    _check_opt(o, c, "frozen_opt_")
    np.testing.assert_array_equal(b.means.cpu().numpy(), c.a("frozen_base_means"))
    np.testing.assert_array_equal(b.log_scales.cpu().numpy(), c.a("frozen_base_log_scales"))


@pytest.mark.parametrize("c", CASES, ids=lambda c: c["name"])
def test_gpu_prune_and_resize(c):
    require_gpu()
    from paper_2604_02851_b200 import pool
    m = _model(c)
    o = _opt(c, m)
    b = _baselines(c)
    removed, rec = pool.prune(m, opacity_floor=0.01)
    np.testing.assert_array_equal(removed, c.a("removed"))
    assert (rec is not None) == c["has_prune"]
    if rec is not None:
        o.resize(rec)
        pool.baselines_apply_record(b, rec)
    _check_model(m, c, "pruned_", c["pruned_active"])
    _check_opt(o, c, "pruned_opt_")
    np.testing.assert_array_equal(b.means.cpu().numpy(), c.a("pruned_base_means"))


@pytest.mark.parametrize("c", CASES, ids=lambda c: c["name"])
def test_gpu_client_append_and_ordering_packet(c):
    require_gpu()
    from paper_2604_02851_b200 import pool
    m = _model(c)
    o = _opt(c, m)
    b = _baselines(c)
    ids = c.a("append_ids")
    rec = pool.AppendRecord(insert_at=c["active"], count=len(ids), object_ids=ids, new_active_count=c["active"] + len(ids))
    pool.apply_mutation(m, rec)
    o.resize(rec)
    pool.baselines_apply_record(b, rec)
    _check_model(m, c, "appended_", c["active"] + len(ids))
    _check_opt(o, c, "appended_opt_")
    np.testing.assert_array_equal(b.means.cpu().numpy(), c.a("appended_base_means"))
    # the tick's ordering packet: [permute?] + append + [prune?]
    recs = []
    if c["has_permute"]:
        recs.append(pool.PermuteRecord(c.a("permutation"), c["frozen_active"]))
    recs.append(rec)
    if c["has_prune"]:
        recs.append(pool.PruneRecord(c.a("removed"), c["pruned_active"]))
    assert pool.encode_ordering(recs) == c.a("packet").tobytes()
