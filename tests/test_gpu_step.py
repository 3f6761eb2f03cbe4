"""GPU optimize step (backward + fp64-moment Adam) vs the reference trajectory.

Tolerances: after each of 3 steps, parameters within 2e-6 absolute of the
reference (Adam's first steps move each coordinate by ~lr*sign(g), so a
gradient that agrees to 1e-6 relative gives the same update up to float32
rounding); the mean loss within 1e-9 (fp64 blend) / 1e-6 (fp32 blend).
"""

import numpy as np
import pytest

from conftest import case_model, load_cases
from gpu_util import require_gpu

pytestmark = pytest.mark.gpu

STEPS = load_cases("step_cases")
GROUPS = ("means", "log_scales", "quaternions", "logit_opacities", "sh_coeffs")


def _setup(c):
    from paper_2604_02851_b200.geometry import CameraIntrinsics, Pose
    from paper_2604_02851_b200.model import GaussianModel
    from paper_2604_02851_b200.optim import OptimizerState, ReferenceView
    from paper_2604_02851_b200.render import LightState
    m = case_model(c, "init_")
    model = GaussianModel(m.means, m.log_scales, m.quaternions, m.logit_opacities, m.sh_coeffs,
                          m.light_visibility, m.object_ids, m.active_count, m.sh_degree)
    light = LightState(c.a("light_dir"), c.a("light_int"), c.a("ambient"))
    light.direction = np.array(c.a("light_dir"))
    intr = CameraIntrinsics(width=c["W"], height=c["H"], fov_y=c["fov"], near=c["near"])
    views = [ReferenceView(Pose(p[:3], p[3:]), intr, gt, light, c.a("bg")) for p, gt in zip(c.a("poses"), c.a("gts"))]
    return model, OptimizerState(model, scene_extent=c["scene_extent"]), views


@pytest.mark.parametrize("c", STEPS, ids=[f"deg{c['degree']}" for c in STEPS])
@pytest.mark.parametrize("precision", [1, 0])
def test_gpu_step_trajectory(c, precision):
    require_gpu()
    from paper_2604_02851_b200.optim import step
    model, state, views = _setup(c)
    for it in range(c["steps"]):
        L = step(model, state, views, precision=precision)
        assert abs(L - c.a("losses")[it]) <= (1e-9 if precision else 1e-6)
        for k in GROUPS:
            np.testing.assert_allclose(getattr(model, k), c.a(f"after{it}_{k}"), rtol=0, atol=2e-6, err_msg=k)
    assert state.step_count == c["steps"]
    np.testing.assert_array_equal(state.age, c.a("age"))
    np.testing.assert_allclose(state.grad_ema, c.a("grad_ema"), rtol=1e-4)
    for k in GROUPS:  # first moments: gradient tolerances of test_gpu_raster (normwise for fp32)
        ref_m = c.a(f"m_{k}")
        err = np.abs(state.m[k] - ref_m)
        assert err.max() <= (2e-6 if precision else 1e-4) * np.abs(ref_m).max(), k
        assert np.linalg.norm(err) <= 1e-4 * np.linalg.norm(ref_m), k


def test_gpu_step_errors_and_noops():
    """ref pkg/tests/test_optim.py:275-302, 386-391."""
    require_gpu()
    from paper_2604_02851_b200.optim import LearningRates, OptimizerState, step
    c = STEPS[0]
    model, state, views = _setup(c)
    before = {k: getattr(model, k).copy() for k in GROUPS}
    # the step renormalises quaternions even at zero LR (optim.py:399), which
    # can move a stored float32 unit quaternion by one ulp
    q = before["quaternions"][: model.active_count].astype(np.float64)
    before["quaternions"][: model.active_count] = (q / np.linalg.norm(q, axis=-1, keepdims=True)).astype(np.float32)
    zero = LearningRates(0, 0, 0, 0, 0, 0)
    s0 = OptimizerState(model, lrs=zero)
    assert step(model, s0, views) > 0
    for k in GROUPS:
        np.testing.assert_array_equal(getattr(model, k), before[k])
    assert s0.step_count == 1
    for v in views:
        v.ready = False
    with pytest.raises(ValueError):
        step(model, state, views)
    for v in views:
        v.ready = True
    model.active_count -= 1
    with pytest.raises(ValueError):
        step(model, state, views)


def test_gpu_step_batch_average():
    """Duplicating a view gives the same update (ref test_optim.py:323-331)."""
    require_gpu()
    from paper_2604_02851_b200.optim import OptimizerState, step
    c = STEPS[0]
    ma, _, views = _setup(c)
    mb = ma.copy()
    step(ma, OptimizerState(ma), [views[0]])
    step(mb, OptimizerState(mb), [views[0], views[0]])
    np.testing.assert_allclose(ma.means, mb.means, atol=1e-7)


@pytest.mark.parametrize("degree", [0, 3])
def test_gpu_deferred_chain_equals_per_view_chain(degree):
    """step()'s deferred chain rule (ss_chain_views: every view in one pass
    over the rows) adds the same fp32 terms in the same order as the
    per-view chain of ss_backward: the gradient is bit-identical, with and
    without a row subset, including rows culled in some views."""
    require_gpu()
    import torch
    from paper_2604_02851_b200 import synth
    from paper_2604_02851_b200.model import DeviceModel
    from paper_2604_02851_b200.optim import StepWorkspace, backward_device, chain_views
    from paper_2604_02851_b200.render import _subset_tensor
    W, H = 256, 144
    host = synth.random_field(40_000, degree, W, H, seed=5)
    host.active_count = 38_000
    dm = DeviceModel.from_host(host, 0)
    tgt = DeviceModel.from_host(synth.target_model(host, seed=6), 0)
    intr = synth.intrinsics(W, H)
    light = synth.light()
    poses = synth.ring_poses(5, radius=1.5)
    from paper_2604_02851_b200.optim import ReferenceView
    from paper_2604_02851_b200.render import render_device
    views = [ReferenceView(p, intr, render_device(tgt, p, intr, light), light, np.zeros(3)) for p in poses]
    rng = np.random.default_rng(0)
    for subset in (None, np.sort(rng.choice(40_000, 25_000, replace=False))):
        sub = _subset_tensor(subset, dm.device)
        ws = StepWorkspace(dm)
        n_grad = dm.active_count * (11 + 3 * (degree + 1) ** 2)
        g_ref = torch.zeros(n_grad, dtype=torch.float32, device=dm.device)
        loss = torch.zeros(1, dtype=torch.float64, device=dm.device)
        for v in views:
            backward_device(dm, v, g_ref, loss, subset_tensor=sub)
        n_in = int(sub.numel()) if sub is not None else dm.count
        g9, rinv = ws.defer_buffers(len(views), n_in, dm.device)
        g_def = torch.zeros_like(g_ref)
        loss2 = torch.zeros(1, dtype=torch.float64, device=dm.device)
        for i, v in enumerate(views):
            backward_device(dm, v, g_def, loss2, subset_tensor=sub, defer=(g9[i], rinv[i]))
        chain_views(dm, views, g9, rinv, g_def, sub)
        assert torch.equal(loss, loss2)
        assert torch.equal(g_ref.view(torch.int32), g_def.view(torch.int32))
        assert bool((g_ref != 0).any())


@pytest.mark.parametrize("degree", [1, 3])
def test_gpu_atomics_mode_matches_deterministic(degree):
    """ss_render_opts.deterministic = 0 (float atomics into the per-row
    screen-space sums, no partials) gives the deterministic mode's gradient
    to fp32 summation-order precision (normwise <= 1e-5 per group) and the
    same loss bit for bit (the loss reduction does not change)."""
    require_gpu()
    import torch
    from paper_2604_02851_b200 import synth
    from paper_2604_02851_b200.model import DeviceModel
    from paper_2604_02851_b200.optim import ReferenceView, backward
    from paper_2604_02851_b200.render import render_device
    W, H = 320, 192
    host = synth.random_field(30_000, degree, W, H, seed=8)
    host.active_count = 29_000
    dm = DeviceModel.from_host(host, 0)
    tgt = DeviceModel.from_host(synth.target_model(host, seed=9), 0)
    intr = synth.intrinsics(W, H)
    light = synth.light()
    pose = synth.ring_poses(3)[1]
    view = ReferenceView(pose, intr, render_device(tgt, pose, intr, light), light, np.zeros(3))
    L0, g0, img0 = backward(dm, view)
    L1, g1, img1 = backward(dm, view, deterministic=False)
    assert L0 == L1
    np.testing.assert_array_equal(img0, img1)
    for k in GROUPS:
        a, b = getattr(g0, k), getattr(g1, k)
        err = np.linalg.norm(a - b) / max(np.linalg.norm(a), 1e-30)
        assert err <= 1e-5, (k, err)
        assert np.linalg.norm(a) > 0


@pytest.mark.parametrize("sync_loss", [False, True])
def test_gpu_sync_free_binning_overflow_recovers(sync_loss):
    """The step bins without reading pair counts back; a step whose pairs
    outgrow the capacity is voided on the device (Adam skipped, sticky) and
    re-run with a larger capacity when its status is checked -- the
    trajectory is bit-identical to a run that never overflowed."""
    require_gpu()
    import torch
    from paper_2604_02851_b200 import _lib, synth
    from paper_2604_02851_b200.model import DeviceModel
    from paper_2604_02851_b200.optim import OptimizerState, ReferenceView, StepWorkspace, step
    from paper_2604_02851_b200.render import render_device
    W, H = 256, 160
    host = synth.random_field(20_000, 2, W, H, seed=21)
    tgt = DeviceModel.from_host(synth.target_model(host, seed=22), 0)
    intr = synth.intrinsics(W, H)
    light = synth.light()
    poses = synth.ring_poses(3, radius=0.5)
    views = [ReferenceView(p, intr, render_device(tgt, p, intr, light), light, np.zeros(3)) for p in poses]
    c = _lib.ctx(0)

    def run(cap):
        dm = DeviceModel.from_host(host, 0)
        state = OptimizerState(dm, scene_extent=2.0)
        ws = StepWorkspace(dm)
        losses = []
        for i in range(4):
            if cap is not None and i in (0, 2):
                _lib.pair_capacity(0, -cap)  # force an overflow at steps 0 and 2
            L = step(dm, state, views, workspace=ws, sync_loss=sync_loss)
            losses.append(float(L) if sync_loss else L)
        ws.flush()
        torch.cuda.synchronize()
        return dm, state, ws

    ref_dm, ref_state, _ = run(None)
    dm, state, ws = run(1000)
    assert state.step_count == ref_state.step_count == 4
    for k in GROUPS:
        assert torch.equal(getattr(dm, k), getattr(ref_dm, k)), k
    np.testing.assert_array_equal(state.age, ref_state.age)
    for k in GROUPS:
        np.testing.assert_array_equal(state.m[k], ref_state.m[k])
    assert int(ws.bins_status[0]) == 0 and not ws.pending
    assert _lib.pair_capacity(0, 0) > 1000


def test_gpu_step_issues_no_host_sync():
    """Once warmed up, optim.step (fp32 path, persistent workspace, device
    loss) enqueues every view's binning, blending, the chain rule and Adam
    without one host synchronisation (ss_host_syncs counts every stream sync,
    read-back and scratch-arena growth the library issues)."""
    require_gpu()
    import torch
    from paper_2604_02851_b200 import _lib, synth
    from paper_2604_02851_b200.model import DeviceModel
    from paper_2604_02851_b200.optim import OptimizerState, ReferenceView, StepWorkspace, step
    from paper_2604_02851_b200.render import render_device
    W, H = 320, 192
    host = synth.random_field(30_000, 3, W, H, seed=31)
    tgt = DeviceModel.from_host(synth.target_model(host, seed=32), 0)
    dm = DeviceModel.from_host(host, 0)
    intr = synth.intrinsics(W, H)
    light = synth.light()
    views = [ReferenceView(p, intr, render_device(tgt, p, intr, light), light, np.zeros(3))
             for p in synth.ring_poses(4, radius=0.5)]
    state = OptimizerState(dm, scene_extent=2.0)
    ws = StepWorkspace(dm)
    for _ in range(3):
        step(dm, state, views, workspace=ws, sync_loss=False)
    ws.flush()
    torch.cuda.synchronize()
    c = _lib.ctx(0)
    before = _lib.host_syncs(0)
    for _ in range(4):
        step(dm, state, views, workspace=ws, sync_loss=False)
    assert _lib.host_syncs(0) == before
    ws.flush()
    assert state.step_count == 7


@pytest.mark.parametrize("lanes", [1, 3])
def test_gpu_view_lanes_bit_identical(lanes, monkeypatch):
    """optim.step deals the views over VIEW_LANES streams (each with its own
    library context); every view's kernels are the same whichever lane runs
    them, so the trajectory is bit-identical to the default (2 lanes)."""
    require_gpu()
    import torch
    from paper_2604_02851_b200 import optim, synth
    from paper_2604_02851_b200.model import DeviceModel
    from paper_2604_02851_b200.optim import OptimizerState, ReferenceView, StepWorkspace, step
    from paper_2604_02851_b200.render import render_device
    W, H = 256, 160
    host = synth.random_field(20_000, 3, W, H, seed=41)
    tgt = DeviceModel.from_host(synth.target_model(host, seed=42), 0)
    intr = synth.intrinsics(W, H)
    light = synth.light()
    views = [ReferenceView(p, intr, render_device(tgt, p, intr, light), light, np.zeros(3))
             for p in synth.ring_poses(5, radius=0.5)]

    def run():
        dm = DeviceModel.from_host(host, 0)
        state = OptimizerState(dm, scene_extent=2.0)
        ws = StepWorkspace(dm)
        losses = [step(dm, state, views, workspace=ws) for _ in range(3)]
        torch.cuda.synchronize()
        return dm, state, losses

    ref_dm, ref_state, ref_l = run()
    monkeypatch.setattr(optim, "VIEW_LANES", lanes)
    dm, state, losses = run()
    assert losses == ref_l
    for k in GROUPS:
        assert torch.equal(getattr(dm, k), getattr(ref_dm, k)), k
    for k in GROUPS:
        np.testing.assert_array_equal(state.m[k], ref_state.m[k])


def test_gpu_step_device_subset_matches_host_subset():
    """index_subset as a CUDA tensor (e.g. pool.precull(..., as_tensor=True),
    unsorted here) gives the same step as the host indices."""
    require_gpu()
    import torch
    from paper_2604_02851_b200 import synth
    from paper_2604_02851_b200.model import DeviceModel
    from paper_2604_02851_b200.optim import OptimizerState, ReferenceView, StepWorkspace, step
    from paper_2604_02851_b200.render import render_device
    W, H = 256, 160
    host = synth.random_field(20_000, 2, W, H, seed=51)
    tgt = DeviceModel.from_host(synth.target_model(host, seed=52), 0)
    intr, light = synth.intrinsics(W, H), synth.light()
    views = [ReferenceView(p, intr, render_device(tgt, p, intr, light), light, np.zeros(3))
             for p in synth.ring_poses(3, radius=0.5)]
    rng = np.random.default_rng(3)
    sub = np.sort(rng.choice(20_000, 14_000, replace=False))

    def run(s):
        dm = DeviceModel.from_host(host, 0)
        state = OptimizerState(dm, scene_extent=2.0)
        ws = StepWorkspace(dm)
        losses = [step(dm, state, views, index_subset=s, workspace=ws) for _ in range(2)]
        torch.cuda.synchronize()
        return dm, losses

    ref_dm, ref_l = run(sub)
    perm = rng.permutation(sub.size)
    dm, losses = run(torch.from_numpy(sub[perm]).cuda())
    assert losses == ref_l
    for k in GROUPS:
        assert torch.equal(getattr(dm, k), getattr(ref_dm, k)), k


def test_gpu_step_repeated_view_object():
    """The same ReferenceView passed twice in one step (its camera's tile
    buffers shared by both backward passes) equals two separate, identical
    view objects."""
    require_gpu()
    import copy
    import torch
    from paper_2604_02851_b200 import synth
    from paper_2604_02851_b200.model import DeviceModel
    from paper_2604_02851_b200.optim import OptimizerState, ReferenceView, StepWorkspace, step
    from paper_2604_02851_b200.render import render_device
    W, H = 256, 160
    host = synth.random_field(20_000, 1, W, H, seed=61)
    tgt = DeviceModel.from_host(synth.target_model(host, seed=62), 0)
    intr, light = synth.intrinsics(W, H), synth.light()
    base = [ReferenceView(p, intr, render_device(tgt, p, intr, light), light, np.zeros(3))
            for p in synth.ring_poses(3, radius=0.5)]

    def run(views):
        dm = DeviceModel.from_host(host, 0)
        state = OptimizerState(dm, scene_extent=2.0)
        ws = StepWorkspace(dm)
        losses = [step(dm, state, views, workspace=ws) for _ in range(3)]
        torch.cuda.synchronize()
        return dm, losses

    a = [base[0], base[1], base[0], base[2], base[0]]
    b = [copy.copy(base[0]), copy.copy(base[1]), copy.copy(base[0]), copy.copy(base[2]), copy.copy(base[0])]
    for v in b:
        v.__dict__.pop("_tile_hint", None), v.__dict__.pop("_tile_order", None)
    dm_a, la = run(a)
    dm_b, lb = run(b)
    assert la == lb
    for k in GROUPS:
        assert torch.equal(getattr(dm_a, k), getattr(dm_b, k)), k
