"""Scene engine on the GPU vs the reference engine.

Expectations are the unmodified reference's own outputs
(tests/golden/make_golden.py::engine_cases: render_ground_truth,
capture_input_buffers, render_depth, render_ortho_depth on scenes with
static and animated planes / spheres / boxes, checker textures and shadows).
The kernel mirrors the reference's float64 arithmetic op for op, including
the FMA pattern of each numpy matmul, so the comparison is exact.
"""

import numpy as np
import pytest

from conftest import load_cases
from gpu_util import require_gpu

CASES = load_cases("engine_cases")
PIN = [c for c in CASES if c["kind"] == "pinhole"]
ORTHO = [c for c in CASES if c["kind"] == "ortho"]
CHANNELS = ("world_pos", "valid", "normal", "albedo", "shaded", "object_id", "depth", "footprint", "lit")


class _Pose:
    """The reference camera frame exactly (position + rotation matrix)."""

    def __init__(self, position, R):
        self.position, self._R = np.asarray(position), np.asarray(R)

    def rotation(self):
        return self._R


def _setup(c):
    from paper_2604_02851_b200.scene import scene_from_dict
    scene = scene_from_dict(c["scene"])
    tf = c.a("transforms")
    tfs = {int(r[0]): (r[1:5], r[5:8]) for r in tf} if len(tf) else None
    return scene, _Pose(c.a("position"), c.a("R")), tfs


def _intr(c):
    from paper_2604_02851_b200.geometry import CameraIntrinsics
    return CameraIntrinsics(width=c["width"], height=c["height"], fov_y=c["fov_y"], near=c["near"], far=c["far"])


def _eq(got, exp, what):
    bad = ~((got == exp) | (np.isnan(got) & np.isnan(exp)) if got.dtype.kind == "f" else (got == exp))
    assert not bad.any(), f"{what}: {int(bad.sum())} of {bad.size} differ, first at {np.argwhere(bad)[:3].tolist()}"


@pytest.mark.gpu
@pytest.mark.parametrize("c", PIN, ids=lambda c: c["name"])
def test_gpu_ground_truth_and_depth_match_reference(c):
    require_gpu()
    from paper_2604_02851_b200 import engine
    scene, pose, tfs = _setup(c)
    intr = _intr(c)
    _eq(engine.render_ground_truth(scene, pose, intr, transforms=tfs), c.a("gt"), "gt")
    _eq(engine.render_depth(scene, pose, intr, transforms=tfs), c.a("render_depth"), "render_depth")
    g32 = engine.render_ground_truth_device(scene, pose, intr, transforms=tfs).cpu().numpy()
    _eq(g32, c.a("gt").astype(np.float32), "gt float32")


@pytest.mark.gpu
@pytest.mark.parametrize("c", PIN, ids=lambda c: c["name"])
def test_gpu_capture_input_buffers_match_reference(c):
    require_gpu()
    from paper_2604_02851_b200 import engine
    scene, pose, tfs = _setup(c)
    b = engine.capture_input_buffers(scene, pose, _intr(c), transforms=tfs)
    for ch in CHANNELS:
        _eq(np.asarray(getattr(b, ch)), c.a(ch), ch)


@pytest.mark.gpu
@pytest.mark.parametrize("c", ORTHO, ids=lambda c: c["name"])
def test_gpu_ortho_depth_matches_reference(c):
    require_gpu()
    from paper_2604_02851_b200 import engine
    from paper_2604_02851_b200.geometry import OrthoCamera
    scene, pose, tfs = _setup(c)
    cam = OrthoCamera(pose=pose, half_width=c["half_width"], half_height=c["half_height"], width=c["width"],
                      height=c["height"], far=c["far"])
    _eq(engine.render_ortho_depth(scene, cam, transforms=tfs), c.a("ortho_depth"), "ortho_depth")


@pytest.mark.gpu
def test_gpu_engine_properties():
    """The reference's own engine tests (pkg/tests/test_scene_engine.py:55-147)
    on the device path: empty scene = background, unlit side = ambient only,
    shadowed floor = albedo * ambient, footprint of a fronto-parallel plane,
    determinism."""
    require_gpu()
    from paper_2604_02851_b200 import engine
    from paper_2604_02851_b200.geometry import CameraIntrinsics, look_at
    from paper_2604_02851_b200.scene import Albedo, DirectionalLight, Plane, SceneDescription, SceneObject
    light = DirectionalLight(direction=[-0.4, -1.0, 0.3], intensity=[0.8, 0.8, 0.8], ambient=[0.2, 0.2, 0.2])
    empty = SceneDescription(objects=(), light=light, background=np.array([0.1, 0.2, 0.3]))
    img = engine.render_ground_truth(empty, look_at([0, 1, -3], [0, 0, 0]), CameraIntrinsics(16, 16, 1.0))
    np.testing.assert_allclose(img, np.broadcast_to([0.1, 0.2, 0.3], (16, 16, 3)))
    up = DirectionalLight(direction=[0, 1, 0], intensity=[1, 1, 1], ambient=[0.25, 0.25, 0.25])
    floor = SceneDescription(objects=(SceneObject(0, Plane([0, 0, 0], [0, 1, 0], (4, 4)), Albedo("solid", [0.6] * 3)),),
                             light=up)
    img = engine.render_ground_truth(floor, look_at([0, 3, 0.01], [0, 0, 0]), CameraIntrinsics(24, 24, 1.2))
    assert (np.abs(img - 0.6 * 0.25).max(axis=-1) < 1e-9).mean() > 0.9
    wall = SceneDescription(objects=(SceneObject(0, Plane([0, 0, 4], [0, 0, -1], (20, 20)), Albedo("solid", [0.5] * 3)),),
                            light=light)
    b = engine.capture_input_buffers(wall, look_at([0, 0, 0], [0, 0, 4]), CameraIntrinsics(4, 256, np.pi / 2))
    assert b.footprint[128, 2] == pytest.approx(0.03125, rel=1e-3)
    a1 = engine.render_ground_truth(floor, look_at([1, 2, 3], [0, 0, 0]), CameraIntrinsics(16, 16, 1.0))
    a2 = engine.render_ground_truth(floor, look_at([1, 2, 3], [0, 0, 0]), CameraIntrinsics(16, 16, 1.0))
    np.testing.assert_array_equal(a1, a2)


@pytest.mark.gpu
def test_gpu_ground_truth_feeds_the_optimiser():
    """A device ground truth drives optim.step without a host round trip."""
    require_gpu()
    import torch
    from paper_2604_02851_b200 import engine, synth
    from paper_2604_02851_b200.geometry import CameraIntrinsics, look_at
    from paper_2604_02851_b200.model import DeviceModel
    from paper_2604_02851_b200.optim import OptimizerState, ReferenceView, step
    from paper_2604_02851_b200.render import LightState
    from paper_2604_02851_b200.scene import scene_from_dict
    c = PIN[0]
    scene = scene_from_dict(c["scene"])
    intr = CameraIntrinsics(64, 48, 1.2)
    pose = look_at([2.5, 2.5, 2.5], [0, 0.3, 0])
    gt = engine.render_ground_truth_device(scene, pose, intr)
    dm = DeviceModel.from_host(synth.random_field(2000, 1, 64, 48, seed=1), 0)
    st = OptimizerState(dm, scene_extent=3.0)
    view = ReferenceView(pose, intr, gt, LightState([-0.4, -1.0, 0.3], [0.8, 0.8, 0.8]), np.zeros(3))
    loss = step(dm, st, [view])
    assert np.isfinite(loss)
    torch.cuda.synchronize()


EXPAND = load_cases("expand_cases")
SAMPLE_FIELDS = ("positions", "normals", "albedo", "object_ids", "footprints", "lit", "camera_indices")
INIT_FIELDS = ("means", "log_scales", "quaternions", "logit_opacities", "sh_coeffs", "light_visibility", "object_ids")


def _buffers(c):
    from paper_2604_02851_b200.engine import InputBuffers

    class _P:
        def __init__(self, position):
            self.position = position

    chans = ("world_pos", "valid", "normal", "albedo", "object_id", "footprint", "lit")
    return [InputBuffers(pose=_P(c.a(f"cam{i}_position")), intrinsics=None, shaded=None, depth=None,
                         **{ch: c.a(f"cam{i}_{ch}") for ch in chans})
            for i in range(c["n_cams"])]


@pytest.mark.gpu
@pytest.mark.parametrize("c", EXPAND, ids=lambda c: c["name"])
def test_gpu_cull_input_samples_matches_reference(c):
    """The reference's own capture buffers in, its SampleBatch out (exact,
    including pool order and the lower-camera tie break)."""
    require_gpu()
    from paper_2604_02851_b200 import engine
    sb = engine.cull_input_samples(_buffers(c))
    assert sb.count == c["kept"]
    for k in SAMPLE_FIELDS:
        _eq(np.asarray(getattr(sb, k)), c.a(f"out_{k}"), k)


@pytest.mark.gpu
@pytest.mark.parametrize("c", EXPAND, ids=lambda c: c["name"])
def test_gpu_init_gaussians_matches_reference(c):
    require_gpu()
    from paper_2604_02851_b200 import engine
    sb = engine.SampleBatch(**{k: c.a(f"out_{k}") for k in SAMPLE_FIELDS})
    for deg in (0, 1):
        g = engine.init_gaussians(sb, sh_degree=deg)
        for k in INIT_FIELDS:
            _eq(np.asarray(getattr(g, k)), c.a(f"init{deg}_{k}"), f"deg{deg} {k}")


# ---- the reference's own engine tests (pkg/tests/test_scene_engine.py:149-300) on the device path

def _light():
    from paper_2604_02851_b200.scene import DirectionalLight
    return DirectionalLight(direction=(-0.4, -1.0, 0.3), intensity=[0.8, 0.8, 0.8], ambient=[0.2, 0.2, 0.2])


def _floor(extra=()):
    from paper_2604_02851_b200.scene import Albedo, Plane, SceneDescription, SceneObject
    objs = [SceneObject(0, Plane([0, 0, 0], [0, 1, 0], (4.0, 4.0)),
                        Albedo("checker", [0.9, 0.9, 0.9], [0.2, 0.25, 0.35], 1.0))] + list(extra)
    return SceneDescription(tuple(objs), _light(), np.array([0.05, 0.05, 0.08]))


def test_dome_rig_degenerate_and_hemisphere():
    from paper_2604_02851_b200.engine import build_dome_rig
    poses, _ = build_dome_rig([1, 0, 2], heading=0.0, n_cameras=1, radius=3.0)
    np.testing.assert_allclose(poses[0].position, [1, 3, 2], atol=1e-12)
    np.testing.assert_allclose(poses[0].forward(), [0, -1, 0], atol=1e-12)
    poses, _ = build_dome_rig([1, 0, 2], heading=0.3, n_cameras=10, radius=3.0)
    for p in poses:
        off = p.position - np.array([1, 0, 2.0])
        assert np.linalg.norm(off) == pytest.approx(3.0) and off[1] >= 0
        np.testing.assert_allclose(p.forward(), -off / np.linalg.norm(off), atol=1e-9)


def test_duplicate_dynamic_ids_rejected():
    from paper_2604_02851_b200.scene import Albedo, SceneDescription, SceneObject, Sphere
    b = SceneObject(3, Sphere([0, 0.5, 0], 0.5), Albedo("solid", [0.8, 0.2, 0.15]))
    with pytest.raises(ValueError):
        SceneDescription((b, b), _light())


@pytest.mark.gpu
def test_gpu_rotating_checker_box_texture_is_rest_frame():
    require_gpu()
    from paper_2604_02851_b200 import engine
    from paper_2604_02851_b200.geometry import CameraIntrinsics, look_at
    from paper_2604_02851_b200.scene import Albedo, Animation, Box, SceneDescription, SceneObject
    box = SceneObject(2, Box([0, 0.5, 0], [0.5, 0.5, 0.5]), Albedo("checker", [1, 1, 1], [0, 0, 0], 0.25),
                      Animation(kind="rotate", axis=[0, 1, 0], deg_per_s=90.0, anchor=[0, 0, 0]))
    scene = SceneDescription((box,), _light())
    pose, intr = look_at([0, 2, -3], [0, 0.5, 0]), CameraIntrinsics(32, 32, 1.0)
    img0 = engine.render_ground_truth(scene, pose, intr, transforms=scene.transforms_at(0.0))
    img4 = engine.render_ground_truth(scene, pose, intr, transforms=scene.transforms_at(4.0))
    img1 = engine.render_ground_truth(scene, pose, intr, transforms=scene.transforms_at(0.5))
    np.testing.assert_allclose(img0, img4, atol=1e-9)
    assert np.abs(img0 - img1).max() > 0.1  # 45 degrees later the pattern moved


@pytest.mark.gpu
def test_gpu_cull_single_identical_and_fronto_parallel():
    require_gpu()
    from paper_2604_02851_b200 import engine
    from paper_2604_02851_b200.geometry import CameraIntrinsics, look_at
    from paper_2604_02851_b200.scene import Albedo, Plane, SceneDescription, SceneObject
    scene = _floor()
    intr = CameraIntrinsics(16, 16, 1.2)
    pose = look_at([0, 3, -3], [0, 0, 0])
    b1 = engine.capture_input_buffers(scene, pose, intr)
    assert engine.cull_input_samples([b1]).count == int(b1.valid.sum())
    b2 = engine.capture_input_buffers(scene, pose, intr)
    batch = engine.cull_input_samples([b1, b2])
    assert batch.count == int(b1.valid.sum()) and (batch.camera_indices == 0).all()
    plane = SceneDescription((SceneObject(0, Plane([0, 0, 0], [0, 1, 0], (3, 3)), Albedo("solid", [0.5] * 3)),), _light())
    intr = CameraIntrinsics(24, 24, 1.2)
    top = engine.capture_input_buffers(plane, look_at([0, 4, 0.01], [0, 0, 0]), intr)
    grazing = engine.capture_input_buffers(plane, look_at([0, 0.3, -4.5], [0, 0, 0]), intr)
    batch = engine.cull_input_samples([grazing, top])  # grazing gets the lower index on purpose
    assert (batch.camera_indices == 1).mean() > 0.95


@pytest.mark.gpu
def test_gpu_ortho_depth_light_camera_and_depth_far():
    require_gpu()
    from paper_2604_02851_b200 import engine
    from paper_2604_02851_b200.geometry import CameraIntrinsics, look_at
    from paper_2604_02851_b200.scene import Albedo, SceneObject, Sphere
    scene = _floor([SceneObject(1, Sphere([0, 0.5, 0], 0.5), Albedo("solid", [0.8, 0.2, 0.15]))])
    cam = engine.build_light_camera([-4, 0, -4], [4, 1, 4], scene.light.direction, resolution=64)
    depth = engine.render_ortho_depth(scene, cam)
    assert depth.shape == (64, 64) and (depth < cam.far).any() and (depth == cam.far).any()
    d = engine.render_depth(_floor(), look_at([0, 2, -4], [0, 0, 4]), CameraIntrinsics(16, 16, 1.2, far=50.0))
    assert (d == 50.0).any() and (d < 50.0).any()


TRACE = [c for c in CASES if c["kind"] == "trace"]


@pytest.mark.gpu
@pytest.mark.parametrize("c", TRACE, ids=lambda c: c["name"])
def test_gpu_trace_and_light_occluded_match_reference(c):
    require_gpu()
    from paper_2604_02851_b200 import engine
    from paper_2604_02851_b200.scene import scene_from_dict
    scene = scene_from_dict(c["scene"])
    tf = c.a("transforms")
    tfs = {int(r[0]): (r[1:5], r[5:8]) for r in tf}
    h = engine.trace(scene, c.a("origins"), c.a("dirs"), tfs)
    for k in ("t", "object_index", "world_point", "normal", "albedo"):
        _eq(np.asarray(getattr(h, k)), c.a(k), k)
    occ = engine.light_occluded(scene, c.a("occ_points"), c.a("occ_normals"), scene.light, tfs)
    _eq(occ, c.a("occluded"), "occluded")
