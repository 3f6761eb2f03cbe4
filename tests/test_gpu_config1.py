"""BASELINE config 1 end to end on the GPU, against the unmodified reference.

Config 1 (BASELINE.json configs[0]): 10k Gaussians, 256x256
views, 4 views per step, 100 optimizer steps, then a full snapshot (profile 0
+ zlib, profile 1), the server's baseline reset from the decoded snapshot, one
more step and one delta tick of every attribute in DELTA_ORDER.  Goldens:
tests/golden/make_config1.py (the reference's own `step`, `encode_snapshot`,
`decode_snapshot` and `StreamServer._emit_delta`).

Trajectories run through the exact path bench.py times (DeviceModel,
StepWorkspace, deferred chain rule, fp32 blend).  The optimisation is
chaotic: a 1e-8 relative perturbation of the loss at step 1 grows ~2.5x per
step (the fp64 blend instantiation, whose gradient buffer is float32 too,
drifts at the same rate), and the reference's own loss curve is not monotone
after ~60 steps.  So the checks are, per SURVEY §8c restated for a chaotic
trajectory:

* free-running, early steps: loss within 1e-5 relative for steps 1-5;
  parameters within 0.01·lr (step 1) and 1·lr (step 10) of their group;
* free-running, 100 steps: the last 20 steps' mean loss within 5 % of the
  reference's; per group, parameters' RMS difference within 2·lr and at most
  0.5 % of the elements beyond 10·lr;
* teacher-forced at step 100: the reference's step-100 model and
  OptimizerState (moments, age, EMA, step count) stepped once on the GPU must
  give the reference's loss within 1e-6 relative and its step-101 parameters
  within 0.05·lr elementwise and 1e-3·lr RMS per group (measured: 0.031·lr and
  2.6e-4·lr): fp32 gradients carry ~1e-6 normwise error, but a small entry can
  be off by ~10 % (cancellation) and Adam's step
  m̂/(√v̂+ε) passes (1-β1)·|Δg|/√v̂ of it into the update;
* the encoders: byte-identical on the reference's own step-100/101 arrays
  and on the GPU run's own arrays (never across runs).
"""

import numpy as np
import pytest

from conftest import load_cases
from gpu_util import require_gpu

pytestmark = pytest.mark.gpu

CASES = load_cases("config1_cases")
TRAIN = ("means", "log_scales", "quaternions", "logit_opacities", "sh_coeffs")
LR = dict(means=2e-4, log_scales=5e-3, quaternions=1e-3, logit_opacities=5e-2)
FRAC_TOL, RMS_TOL = 5e-3, 2.0


def _setup(c):
    import torch
    from paper_2604_02851_b200.geometry import CameraIntrinsics, Pose
    from paper_2604_02851_b200.model import DeviceModel, GaussianModel
    from paper_2604_02851_b200.optim import OptimizerState, ReferenceView, StepWorkspace
    from paper_2604_02851_b200.render import LightState
    g = lambda k: np.array(c.a("init_" + k))
    model = GaussianModel(g("means"), g("log_scales"), g("quaternions"), g("logit_opacities"), g("sh_coeffs"),
                          g("light_visibility"), g("object_ids"), c["n"], c["degree"])
    dm = DeviceModel.from_host(model)
    li = c["light"]
    light = LightState(li["direction"], li["intensity"], np.array(li["ambient"]))
    light.direction = np.array(li["direction"], np.float64)
    intr = CameraIntrinsics(width=c["W"], height=c["H"], fov_y=c["fov"], near=c["near"])
    views = [ReferenceView(Pose(p[:3], p[3:]), intr, torch.from_numpy(gt).cuda(), light, np.array(c["bg"]))
             for p, gt in zip(c.a("poses"), c.a("gts"))]
    state = OptimizerState(dm, scene_extent=c["scene_extent"])
    return dm, state, views, StepWorkspace(dm)


def _lr(c, k):
    if k == "means":
        return LR[k] * c["scene_extent"]
    return LR.get(k)


def _param_stats(c, dm, s):
    """Per group: (max, rms, fraction > 10) of |GPU - reference| in units of the group's lr."""
    out = {}
    for k in TRAIN:
        got = getattr(dm, k).cpu().numpy().astype(np.float64)
        ref = c.a(f"s{s}_{k}").astype(np.float64)
        if k == "sh_coeffs":
            parts = (("sh_dc", got[:, :, :1], ref[:, :, :1], 2.5e-3), ("sh_rest", got[:, :, 1:], ref[:, :, 1:], 1.25e-4))
        else:
            parts = ((k, got, ref, _lr(c, k)),)
        for name, a, b, lr in parts:
            if a.size == 0:
                continue
            d = np.abs(a - b) / lr
            out[name] = (float(d.max()), float(np.sqrt(np.mean(d * d))), float(np.mean(d > 10.0)))
            print(f"deg {c['degree']} step {s} {name}: max {out[name][0]:.3g} lr, rms {out[name][1]:.3g} lr, "
                  f"frac>10lr {out[name][2]:.2e}")
    return out


def _check_params(c, dm, s, frac_tol=FRAC_TOL, rms_tol=RMS_TOL):
    for name, (_, rms, outside) in _param_stats(c, dm, s).items():
        assert outside <= frac_tol, (name, s, outside)
        assert rms <= rms_tol, (name, s, rms)


@pytest.mark.parametrize("c", CASES, ids=[f"deg{c['degree']}" for c in CASES])
def test_config1_trajectory_fp32_bench_path(c):
    """100 steps + the post-snapshot step through the bench's step() path."""
    require_gpu()
    from paper_2604_02851_b200.optim import step
    dm, state, views, ws = _setup(c)
    ref_losses = c.a("losses")
    losses, stats = [], {}
    for s in range(1, c["steps"] + 2):
        losses.append(step(dm, state, views, workspace=ws))
        if s in c["checkpoints"]:
            stats[s] = _param_stats(c, dm, s)
    losses = np.array(losses)
    rel = np.abs(losses - ref_losses) / ref_losses
    print(f"deg {c['degree']} loss rel err per step: " + " ".join(f"{x:.1e}" for x in rel[:12]) + " ...")
    late = abs(losses[80:100].mean() / ref_losses[80:100].mean() - 1)
    print(f"deg {c['degree']} steps 81-100 mean loss {losses[80:100].mean():.6f} vs {ref_losses[80:100].mean():.6f}"
          f" ({late:.2%})")
    assert rel[:5].max() <= 1e-5
    assert late <= 0.05
    for name, (mx, _, _) in stats[1].items():
        assert mx <= 0.01, (name, 1, mx)
    for name, (mx, _, _) in stats[10].items():
        assert mx <= 1.0, (name, 10, mx)
    for s in (100, 101):
        for name, (_, rms, outside) in stats[s].items():
            assert outside <= FRAC_TOL, (name, s, outside)
            assert rms <= RMS_TOL, (name, s, rms)
    assert state.step_count == c["steps"] + 1
    assert (state.age == c["steps"] + 1).all()


@pytest.mark.parametrize("c", CASES, ids=[f"deg{c['degree']}" for c in CASES])
def test_config1_teacher_forced_step_101(c):
    """The reference's step-100 model and optimizer state, one GPU step."""
    require_gpu()
    import torch
    from paper_2604_02851_b200.optim import step
    dm, state, views, ws = _setup(c)
    for k in TRAIN:
        getattr(dm, k).copy_(torch.from_numpy(np.array(c.a(f"s100_{k}"))))
        state.m[k][...] = c.a(f"m100_{k}")
        state.v[k][...] = c.a(f"v100_{k}")
    state.age[...] = c.a("age100")
    state.grad_ema[...] = c.a("ema100")
    state.step_count = c["steps"]
    L = step(dm, state, views, workspace=ws)
    ref_L = c.a("losses")[c["steps"]]
    print(f"deg {c['degree']} teacher-forced step 101: loss rel err {abs(L / ref_L - 1):.2e}")
    assert abs(L / ref_L - 1) <= 1e-6
    for name, (mx, rms, _) in _param_stats(c, dm, c["steps"] + 1).items():
        assert mx <= 0.05, (name, mx)
        assert rms <= 1e-3, (name, rms)


@pytest.mark.parametrize("c", CASES[:1], ids=[f"deg{c['degree']}" for c in CASES[:1]])
def test_config1_trajectory_fp64_blend(c):
    """The fp64 blend instantiation over the first 5 steps."""
    require_gpu()
    from paper_2604_02851_b200.optim import step
    dm, state, views, ws = _setup(c)
    ref_losses = c.a("losses")
    for s in range(1, 6):
        L = step(dm, state, views, workspace=ws, precision=1)
        print(f"fp64 blend step {s}: loss rel err {abs(L / ref_losses[s - 1] - 1):.2e}")
        assert abs(L - ref_losses[s - 1]) <= 1e-6 * ref_losses[s - 1]


@pytest.mark.parametrize("c", CASES, ids=[f"deg{c['degree']}" for c in CASES])
def test_config1_snapshot_reset_and_tick_bytes(c):
    """encode_snapshot (p0 zlib, p1), the decoded-baseline reset, and the
    DELTA_ORDER tick on the reference's own arrays: byte-identical."""
    require_gpu()
    import torch
    from paper_2604_02851_b200.model import DeviceModel, GaussianModel
    from paper_2604_02851_b200.protocol import (PROFILE_DEFAULT, PROFILE_LOSSLESS, DeltaEmitter, DeviceBaselines,
                                                encode_snapshot)
    g100 = {k: np.array(c.a(f"s100_{k}")) for k in TRAIN}
    fixed = {k: np.array(c.a("init_" + k)) for k in ("light_visibility", "object_ids")}
    m100 = GaussianModel(**g100, **fixed, active_count=c["n"], sh_degree=c["degree"])
    p0, (bm, bl) = encode_snapshot(m100, PROFILE_DEFAULT, return_baselines=True)
    assert p0 == c.a("snap_p0").tobytes()
    assert encode_snapshot(m100, PROFILE_LOSSLESS) == c.a("snap_p1").tobytes()
    np.testing.assert_array_equal(bm, c.a("base_means"))
    np.testing.assert_array_equal(bl, c.a("base_log_scales"))

    g101 = {k: np.array(c.a(f"s101_{k}")) for k in TRAIN}
    dm = DeviceModel.from_host(GaussianModel(**g101, **fixed, active_count=c["n"], sh_degree=c["degree"]))
    base = DeviceBaselines(torch.from_numpy(bm).cuda(), torch.from_numpy(bl).cuda(), 1)
    out = DeltaEmitter(dm, base, compression_id=1).tick(0)
    assert [a for a, _ in out] == c["tick_attrs"]
    for a, payload in out:
        assert payload == c.a(f"tick_{a}").tobytes(), a
    np.testing.assert_array_equal(base.means.cpu().numpy(), c.a("tick_base_means"))
    np.testing.assert_array_equal(base.log_scales.cpu().numpy(), c.a("tick_base_log_scales"))


@pytest.mark.parametrize("c", CASES, ids=[f"deg{c['degree']}" for c in CASES])
def test_config1_encoders_on_gpu_run_arrays(c):
    """The GPU run's own step-100 model: snapshot and the next tick equal the
    oracle's encoders on the same arrays (never across runs)."""
    require_gpu()
    import torch
    from oracle import codec as oc
    from paper_2604_02851_b200.optim import step
    from paper_2604_02851_b200.protocol import PROFILE_DEFAULT, DeltaEmitter, DeviceBaselines, encode_snapshot
    dm, state, views, ws = _setup(c)
    for _ in range(20):
        step(dm, state, views, workspace=ws, sync_loss=False)
    host = dm.to_host()
    p0, (bm, bl) = encode_snapshot(dm, PROFILE_DEFAULT, return_baselines=True)
    ref0 = oc.snapshot_payload(host.means, host.log_scales, host.quaternions, host.logit_opacities,
                               host.sh_coeffs, host.light_visibility, host.object_ids, host.active_count,
                               host.sh_degree, 0, 1)
    assert p0 == ref0
    step(dm, state, views, workspace=ws)
    host = dm.to_host()
    base = DeviceBaselines(torch.from_numpy(bm).cuda(), torch.from_numpy(bl).cuda(), 1)
    out = DeltaEmitter(dm, base, compression_id=0).tick(0)
    rb_m, rb_l = bm.copy(), bl.copy()
    a = c["n"]
    for attr, payload in out:
        if attr == 0:
            ref, rb_m = oc.delta_payload(0, host.means[:a], rb_m[:a], None, 0)
        elif attr == 1:
            ref, rb_l = oc.delta_payload(1, host.log_scales[:a], rb_l[:a], None, 0)
        elif attr == 2:
            ref, _ = oc.delta_payload(2, host.quaternions[:a], None, None, 0)
        elif attr == 3:
            ref, _ = oc.delta_payload(3, host.logit_opacities[:a], None, None, 0)
        elif attr == 4:
            ref, _ = oc.delta_payload(4, host.sh_coeffs[:a, :, 0], None, None, 0)
        else:
            ref, _ = oc.delta_payload(5, host.sh_coeffs[:a, :, 1:], None, None, 0)
        assert payload == ref, attr
    np.testing.assert_array_equal(base.means.cpu().numpy(), rb_m)
    np.testing.assert_array_equal(base.log_scales.cpu().numpy(), rb_l)
