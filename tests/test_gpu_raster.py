"""GPU rasterizer vs the oracle and the reference's golden vectors.

Bit-exact: depth order, pixel windows, tile lists / tile ranges (vs oracle,
which mirrors the kernel's fp64 op order), and the reference's own windows /
order.  Tolerances (stated per SURVEY.md §8c):
  fp64 blend (precision=1): image |d| <= 1e-10; gradients within 2e-6 of the
      largest entry per group (the gradient buffer is float32).
  fp32 blend (precision=0): image max|d| <= 1e-4, mean|d| <= 1e-6; gradients
      normwise ||d||/||g|| <= 1e-4 and max|d| <= 1e-4 * max|g| per group.
"""

import numpy as np
import pytest

from conftest import load_cases
from gpu_util import oracle_args, product_args, require_gpu
from oracle import raster as orr

pytestmark = pytest.mark.gpu

RASTER = load_cases("raster_cases")
GROUPS = ("means", "log_scales", "quaternions", "logit_opacities", "sh_coeffs")


def _subset(c):
    return c.a("subset") if c.has("subset") else None


@pytest.mark.parametrize("c", RASTER, ids=[c["name"] for c in RASTER])
def test_gpu_prepare_matches_reference_and_oracle(c):
    require_gpu()
    from paper_2604_02851_b200.render import prepare_splats
    model, pose, intr, light = product_args(c)
    p = prepare_splats(model, pose, intr, light, _subset(c), c["cutoff"])
    np.testing.assert_array_equal(p.rows, c.a("rows"))
    np.testing.assert_array_equal(p.order, c.a("order"))
    np.testing.assert_array_equal(p.windows, c.a("windows"))
    om, cam, ol = oracle_args(c, pose, intr)
    o = orr.prepare(om, cam, ol, _subset(c), c["cutoff"])
    np.testing.assert_array_equal(p.depth, o["depth"])           # bit-exact vs oracle
    np.testing.assert_array_equal(p.windows, o["rect"])
    np.testing.assert_array_equal(p.radius, o["radius"])
    np.testing.assert_array_equal(p.mu2d, o["mu2d"])
    np.testing.assert_array_equal(p.Sigma2d, o["Sigma2d"])
    np.testing.assert_allclose(p.color_pre, c.a("color_pre"), rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(p.opacity, c.a("opacity"), rtol=1e-14)
    np.testing.assert_allclose(p.shade_inter["s"], c.a("s"), rtol=1e-12, atol=1e-13)


@pytest.mark.parametrize("c", RASTER, ids=[c["name"] for c in RASTER])
def test_gpu_tile_bins_bit_exact(c):
    require_gpu()
    from paper_2604_02851_b200.render import tile_bins
    model, pose, intr, light = product_args(c)
    rows, ranges, ranks = tile_bins(model, pose, intr, _subset(c), c["cutoff"])
    om, cam, ol = oracle_args(c, pose, intr)
    o = orr.tile_bins(orr.prepare(om, cam, ol, _subset(c), c["cutoff"]), c["W"], c["H"])
    np.testing.assert_array_equal(rows, o["order_rows"])
    np.testing.assert_array_equal(ranges, o["ranges"])
    np.testing.assert_array_equal(ranks, o["pair_rank"])


@pytest.mark.parametrize("c", RASTER, ids=[c["name"] for c in RASTER])
@pytest.mark.parametrize("precision", [1, 0])
def test_gpu_render(c, precision):
    require_gpu()
    from paper_2604_02851_b200.render import render
    model, pose, intr, light = product_args(c)
    img, T = render(model, pose, intr, light, _subset(c), c.a("bg"), True, c["cutoff"], precision)
    d = np.abs(img - c.a("image"))
    dT = np.abs(T - c.a("T"))
    if precision == 1:
        assert d.max(initial=0) <= 1e-10 and dT.max(initial=0) <= 1e-10
    else:
        assert d.max(initial=0) <= 1e-4 and d.mean() <= 1e-6, (d.max(), d.mean())
        assert dT.max(initial=0) <= 1e-4


@pytest.mark.parametrize("c", RASTER, ids=[c["name"] for c in RASTER])
@pytest.mark.parametrize("precision", [1, 0])
def test_gpu_backward(c, precision):
    require_gpu()
    from paper_2604_02851_b200.optim import ReferenceView, backward
    model, pose, intr, light = product_args(c)
    view = ReferenceView(pose, intr, c.a("gt"), light, c.a("bg"))
    L, g, img = backward(model, view, _subset(c), c["cutoff"], precision)
    tol = 1e-10 if precision else 1e-4
    assert np.abs(img - c.a("image")).max(initial=0) <= tol
    assert abs(L - c["loss"]) <= (1e-12 if precision else 1e-6)
    for name in GROUPS:
        ref = c.a(f"g_{name}")
        got = getattr(g, name)
        assert got.shape == ref.shape, name
        scale = np.abs(ref).max(initial=0.0)
        err = np.abs(got - ref)
        if scale == 0:
            assert err.max(initial=0) == 0, name
            continue
        if precision:
            assert err.max() <= 2e-6 * scale, (name, err.max() / scale)
        else:
            assert np.linalg.norm(err) <= 1e-4 * np.linalg.norm(ref), (name, np.linalg.norm(err) / np.linalg.norm(ref))
            assert err.max() <= 1e-4 * scale, (name, err.max() / scale)


def test_gpu_capped_alpha_and_behind_camera_exact_zeros():
    """ref pkg/tests/test_optim.py:173-228: masked paths are exact zeros."""
    require_gpu()
    from paper_2604_02851_b200.optim import ReferenceView, backward
    c = [c for c in RASTER if c["name"] == "capped"][0]
    model, pose, intr, light = product_args(c)
    view = ReferenceView(pose, intr, c.a("gt"), light, c.a("bg"))
    for prec in (0, 1):
        _, g, _ = backward(model, view, None, True, prec)
        ref = c.a("g_log_scales")
        np.testing.assert_array_equal(g.log_scales[ref == 0.0], 0.0)
    c = [c for c in RASTER if c["name"] == "frozen_tail"][0]
    model, pose, intr, light = product_args(c)
    view = ReferenceView(pose, intr, c.a("gt"), light, c.a("bg"))
    _, g, _ = backward(model, view, None, True, 0)
    for name in GROUPS:
        assert np.all(getattr(g, name)[5] == 0.0)  # row 5 is behind the camera


def test_gpu_backward_deterministic():
    require_gpu()
    from paper_2604_02851_b200.optim import ReferenceView, backward
    c = [c for c in RASTER if c["name"] == "medium"][0]
    model, pose, intr, light = product_args(c)
    view = ReferenceView(pose, intr, c.a("gt"), light, c.a("bg"))
    a = backward(model, view)
    b = backward(model, view)
    assert a[0] == b[0]
    np.testing.assert_array_equal(a[2], b[2])
    for name in GROUPS:
        np.testing.assert_array_equal(getattr(a[1], name), getattr(b[1], name))


def test_gpu_depth_order_exact_at_scale_with_near_ties():
    """300k Gaussians over a 3 m depth range (the 32-bit sort key drops ~21
    low bits there) plus planted depth ties and 1-ulp neighbours: the composite
    order must still equal the exact lexsort((rows, depth)) of the oracle."""
    require_gpu()
    from paper_2604_02851_b200 import synth
    from paper_2604_02851_b200.render import tile_bins
    model = synth.random_field(300_000, 1, 640, 360, seed=11)
    z = model.means[:, 2]
    z[1000:1100] = z[0]                                   # exact ties
    z[2000:2050] = np.nextafter(z[3000], np.float32(10))  # 1-ulp (float32) neighbours
    z[2050:2100] = z[3000]
    intr = synth.intrinsics(640, 360)
    pose = synth.ring_poses(4)[0]
    rows, ranges, ranks = tile_bins(model, pose, intr)
    cam = orr.camera(pose, intr)
    light = dict(direction=np.array([0.0, -1.0, 0.0]), intensity=np.zeros(3), ambient=None)
    o = orr.prepare(model, cam, light)
    np.testing.assert_array_equal(rows, o["rows"][o["order"]])
    b = orr.tile_bins(o, 640, 360)
    np.testing.assert_array_equal(ranges, b["ranges"])
    np.testing.assert_array_equal(ranks, b["pair_rank"])


def test_gpu_long_tile_lists():
    """Tiles holding thousands of splats: 9000 Gaussians on a 40x24 frame
    (6 tiles), with planted depth ties; lists, ranges and ranks equal the
    oracle's exact order."""
    require_gpu()
    from paper_2604_02851_b200 import synth
    from paper_2604_02851_b200.render import tile_bins
    model = synth.random_field(9000, 1, 40, 24, seed=21)
    z = model.means[:, 2]
    z[100:400] = z[0]
    intr = synth.intrinsics(40, 24)
    pose = synth.ring_poses(4)[1]
    rows, ranges, ranks = tile_bins(model, pose, intr)
    cam = orr.camera(pose, intr)
    light = dict(direction=np.array([0.0, -1.0, 0.0]), intensity=np.zeros(3), ambient=None)
    o = orr.prepare(model, cam, light)
    b = orr.tile_bins(o, 40, 24)
    assert (np.diff(b["ranges"], axis=1).max()) > 2048
    np.testing.assert_array_equal(rows, o["rows"][o["order"]])
    np.testing.assert_array_equal(ranges, b["ranges"])
    np.testing.assert_array_equal(ranks, b["pair_rank"])


COMPOSITE = load_cases("composite_cases")


@pytest.mark.gpu
@pytest.mark.parametrize("c", COMPOSITE, ids=lambda c: c["name"])
def test_gpu_composite_of_reference_prepared_splats(c):
    """render.composite on the reference's own PreparedSplats (as prepared,
    and with edited opacity / colour / draw order / infinite radii) equals the
    reference's composite: image and transmittance within the fp64 blend
    tolerance (the only differences are exp's last bits)."""
    require_gpu()
    from types import SimpleNamespace
    from paper_2604_02851_b200.geometry import CameraIntrinsics
    from paper_2604_02851_b200.render import composite
    prep = SimpleNamespace(**{k: c.a(k) for k in ("order", "mu2d", "radius", "inv2d", "opacity", "color")})
    intr = CameraIntrinsics(width=c["W"], height=c["H"], fov_y=1.0)
    img, T = composite(prep, intr, np.array([0.1, 0.2, 0.3]))
    np.testing.assert_allclose(img, c.a("img"), rtol=0, atol=1e-9)
    np.testing.assert_allclose(T, c.a("T"), rtol=0, atol=1e-9)


def test_gpu_render_device_many_matches_single():
    """render_device_many (viewpoints over 3 lanes of streams, one library
    context each, 2 output buffers) == render_device per viewpoint, bit for bit."""
    require_gpu()
    import torch
    from paper_2604_02851_b200 import synth
    from paper_2604_02851_b200.model import DeviceModel
    from paper_2604_02851_b200.render import render_device, render_device_many
    W, H = 320, 192
    m = DeviceModel.from_host(synth.random_field(40_000, 3, W, H, seed=8), 0)
    intr, light = synth.intrinsics(W, H), synth.light()
    poses = synth.ring_poses(7, radius=0.6)
    ref = [render_device(m, p, intr, light).clone() for p in poses]
    got = [g.clone() for g in render_device_many(m, poses, intr, light, lanes=3)]
    for a, b in zip(ref, got):
        assert torch.equal(a, b)
    outs = [torch.empty((H, W, 3), dtype=torch.float32, device=m.device) for _ in range(3)]
    last = render_device_many(m, poses[:3], intr, light, outs=outs, lanes=3)
    torch.cuda.synchronize()
    for a, b in zip(ref[:3], last):
        assert torch.equal(a, b)


def test_gpu_evaluated_pairs_counter_matches_oracle():
    """the roofline's work count -- (pixel, splat) evaluations
    that pass the T-gate, counted by the forward kernel in timing runs --
    against the oracle's own count on a config-1-sized view (10k Gaussians,
    256x256).  fp32 vs fp64 may flip the T-gate of a handful of pixels."""
    require_gpu()
    from oracle import raster as orr
    from paper_2604_02851_b200 import _lib, synth
    from paper_2604_02851_b200.model import DeviceModel
    from paper_2604_02851_b200.render import render_device
    W = H = 256
    host = synth.random_field(10_000, 3, W, H, seed=5)
    dm = DeviceModel.from_host(host, 0)
    intr, light = synth.intrinsics(W, H), synth.light()
    pose = synth.ring_poses(4, radius=0.5)[1]
    c = _lib.ctx(0)
    render_device(dm, pose, intr, light)  # warm (no counting)
    _lib.set_timing(c, True)
    _lib.get_timing(c, reset=True)
    render_device(dm, pose, intr, light)
    _, counters = _lib.get_timing(c, reset=True)
    _lib.set_timing(c, False)
    cam = orr.camera(pose, intr)
    olight = dict(direction=light.direction, intensity=light.intensity, ambient=light.ambient_sh)
    prep = orr.prepare(host, cam, olight, None, True)
    _, _, pairs = orr.composite(prep, W, H, np.zeros(3))
    assert pairs > 100_000
    assert abs(int(counters[0]) - pairs) <= max(10, 1e-5 * pairs), (int(counters[0]), pairs)
