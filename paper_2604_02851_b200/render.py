"""Forward renderer API on the B200 rasterizer.

Drop-in for ref pkg/src/splatstream/render.py: LightState (render.py:34),
flat_ambient_sh (render.py:51), prepare_splats (render.py:226), render
(render.py:339), update_light_visibility (render.py:350).  The compute runs in
libsplat_b200.so (K1-K5, see csrc/ss_raster.cu); this module only marshals
arguments.  `precision=1` selects the fp64 blend instantiation used for
verbatim parity; the default fp32 blend is the throughput path.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from .geometry import quat_to_rotmat
from .model import DeviceModel, as_device

SH_C0 = 0.2820947918
TRANSMITTANCE_CUTOFF = 1e-4
ALPHA_CAP = 0.999
COV2D_BLUR = 0.3


@dataclass
class LightState:
    direction: np.ndarray
    intensity: np.ndarray
    ambient_sh: Optional[np.ndarray] = None

    def __post_init__(self):
        d = np.asarray(self.direction, dtype=np.float64)
        self.direction = d / np.linalg.norm(d)
        self.intensity = np.asarray(self.intensity, dtype=np.float64)
        if self.ambient_sh is not None:
            self.ambient_sh = np.asarray(self.ambient_sh, dtype=np.float64)


def flat_ambient_sh(ambient_rgb) -> np.ndarray:
    return (SH_C0 * np.asarray(ambient_rgb, np.float64))[:, None]


def light_state_from_scene(light) -> LightState:
    """ref render.py:58-60: the scene's directional light with its flat ambient term."""
    return LightState(direction=light.direction, intensity=light.intensity, ambient_sh=flat_ambient_sh(light.ambient))


def camera_struct(pose, intr) -> _lib.SSCamera:
    c = _lib.SSCamera()
    c.position = _lib.f64arr(pose.position, 3)
    R = pose.rotation() if hasattr(pose, "rotation") else quat_to_rotmat(pose.quaternion)
    c.rot_cw = _lib.f64arr(np.asarray(R, np.float64).ravel(), 9)
    fy = (intr.height / 2.0) / np.tan(intr.fov_y / 2.0)
    c.fx, c.fy = float(fy), float(fy)
    c.cx, c.cy = intr.width / 2.0, intr.height / 2.0
    c.near_plane = float(intr.near)
    c.width, c.height = int(intr.width), int(intr.height)
    return c


def light_struct(light) -> _lib.SSLight:
    s = _lib.SSLight()
    s.direction = _lib.f64arr(light.direction, 3)
    s.intensity = _lib.f64arr(light.intensity, 3)
    amb = getattr(light, "ambient_sh", None)
    if amb is None:
        s.ambient_bands = 0
    else:
        amb = np.asarray(amb, np.float64)
        if amb.ndim != 2 or amb.shape[0] != 3 or amb.shape[1] > 16:
            raise ValueError("ambient SH must be (3, bands<=16)")
        s.ambient_bands = amb.shape[1]
        s.ambient = _lib.f64arr(amb.ravel(), 48)
    return s


def _subset_tensor(index_subset, device):
    """The row subset as a sorted device int64 tensor (composite ties break
    by row, render.py:283).  A CUDA tensor is sorted in place on the device;
    host indices go up through pinned memory without a host stall (a
    pageable upload would wait for all the work queued before it)."""
    if index_subset is None:
        return None
    import torch
    if isinstance(index_subset, torch.Tensor) and index_subset.is_cuda:
        t = index_subset.to(device=device, dtype=torch.int64).reshape(-1)
        return torch.sort(t).values
    idx = np.sort(np.asarray(index_subset, np.int64).ravel())
    return torch.from_numpy(idx).pin_memory().to(device, non_blocking=True)


def render_opts(background, subset, extent_cutoff, precision, deterministic=1, gt_ready=None,
                tile_hint=None, defer=None, tile_order=None, bins_status=None) -> _lib.SSRenderOpts:
    o = _lib.SSRenderOpts()
    o.gt_ready = gt_ready
    if bins_status is not None:  # sync-free binning (see ss_render_opts.bins_status)
        o.bins_status = bins_status.data_ptr()
    if tile_order is not None:  # (buffer, valid): the backward's walk order, reused by the next forward
        o.tile_order, o.tile_order_valid = tile_order[0].data_ptr(), int(bool(tile_order[1]))
    if defer is not None:  # (g9, rinv) device buffers: the chain rule is deferred to ss_chain_views
        o.defer_g9, o.defer_rinv = defer[0].data_ptr(), defer[1].data_ptr()
    if tile_hint is not None:
        o.tile_hint = tile_hint.data_ptr()
        o.tile_hint_len = int(tile_hint.numel())
    o.background = _lib.f64arr(background, 3)
    o.subset = subset.data_ptr() if subset is not None else None
    o.subset_count = int(subset.numel()) if subset is not None else 0
    o.extent_cutoff = 1 if extent_cutoff else 0
    o.precision = int(precision)
    o.deterministic = int(deterministic)
    return o


def render_device(model: DeviceModel, pose, intr, light_state, index_subset=None, background=(0.0, 0.0, 0.0),
                  return_transmittance=False, extent_cutoff=True, precision=0, out=None):
    """render() with the image left in HBM: returns a torch (H,W,3) tensor
    (float32, or float64 for precision=1) [and T (H,W)]."""
    import torch
    c = _lib.ctx(model.device.index)
    dt = torch.float64 if precision else torch.float32
    H, W = intr.height, intr.width
    img = out if out is not None else torch.empty((H, W, 3), dtype=dt, device=model.device)
    T = torch.empty((H, W), dtype=dt, device=model.device) if return_transmittance else None
    sub = _subset_tensor(index_subset, model.device)
    m = model.struct()
    cam = camera_struct(pose, intr)
    L = light_struct(light_state)
    o = render_opts(background, sub, extent_cutoff, precision)
    st = _lib.SSRenderStats()
    c.check(c.lib.ss_render(c.handle, m, cam, L, o, _lib.ptr(img), _lib.ptr(T), st))
    return (img, T) if return_transmittance else img


def render_device_many(model: DeviceModel, poses, intr, light_state, outs=None, lanes: int = 4,
                       background=(0.0, 0.0, 0.0), extent_cutoff=True):
    """render_device() of several viewpoints (the client-viewpoint serving
    path), dealt over `lanes` streams with one library
    context each so one viewpoint's latency-bound binning overlaps another's
    blend; the caller's stream waits for all of them.  `outs`: optional
    (H, W, 3) float32 output buffers, one per lane (lane k writes outs[k];
    with fewer buffers than lanes the lane count drops to the buffer count).
    Returns the images in pose order (with `outs`, a buffer holds the last
    image its lane wrote)."""
    import torch
    dev = model.device
    cur = torch.cuda.current_stream(dev)
    L = max(1, int(lanes))
    if outs:
        L = min(L, len(outs))
    streams = [cur] + [_lib.lane_stream(dev.index, k) for k in range(1, L)]
    for s in streams[1:]:
        s.wait_stream(cur)
    H, W = intr.height, intr.width
    m = model.struct()
    L_ = light_struct(light_state)
    o = render_opts(background, None, extent_cutoff, 0)
    imgs = []
    for i, pose in enumerate(poses):
        k = i % L
        with torch.cuda.stream(streams[k]):
            c = _lib.lane_ctx(dev.index, k)
            # lane k always writes outs[k]: its images are ordered on its stream
            img = outs[k] if outs else torch.empty((H, W, 3), dtype=torch.float32, device=dev)
            st = _lib.SSRenderStats()
            c.check(c.lib.ss_render(c.handle, m, camera_struct(pose, intr), L_, o, _lib.ptr(img), None, st))
            imgs.append(img)
    for s in streams[1:]:
        cur.wait_stream(s)
    if not outs:  # allocated on lane streams, handed to the caller's stream
        for img in imgs:
            img.record_stream(cur)
    return imgs


def render(model, pose, intr, light_state, index_subset=None, background=(0.0, 0.0, 0.0),
           return_transmittance: bool = False, extent_cutoff: bool = True, precision: int = 0):
    """ref render.py:339 -- returns a float64 numpy image [, T]."""
    dm, _ = as_device(model, keep_f64=precision == 1)
    r = render_device(dm, pose, intr, light_state, index_subset, background, return_transmittance, extent_cutoff,
                      precision)
    if return_transmittance:
        return r[0].double().cpu().numpy(), r[1].double().cpu().numpy()
    return r.double().cpu().numpy()


@dataclass
class PreparedSplats:
    """Host view of the per-splat preprocess, every field of ref
    render.py:200-223 (model-row order; `order` is the composite order)."""

    rows: np.ndarray
    mu_cam: np.ndarray
    depth: np.ndarray
    mu2d: np.ndarray
    J: np.ndarray
    W: np.ndarray
    Sigma3d: np.ndarray
    cov_cam: np.ndarray
    Sigma2d: np.ndarray
    inv2d: np.ndarray
    opacity: np.ndarray
    color: np.ndarray
    color_pre: np.ndarray
    view_dir: np.ndarray
    view_dist: np.ndarray
    n_hat: np.ndarray
    n_axis: np.ndarray
    shade_inter: dict
    order: np.ndarray
    radius: np.ndarray
    windows: np.ndarray = None


def prepare_splats(model, pose, intr, light_state, index_subset=None, extent_cutoff: bool = True) -> PreparedSplats:
    """ref render.py:226 -- computed by the fp64 preprocess kernel (K1), the
    depth sort (K3a) and ss_prepare_extras (the remaining PreparedSplats
    fields, same device functions); returned as host arrays."""
    import torch
    dm, _ = as_device(model, keep_f64=True)
    c = _lib.ctx(dm.device.index)
    dev = dm.device
    sub = _subset_tensor(index_subset, dev)
    n = int(sub.numel()) if sub is not None else dm.count
    cap = max(n, 1)
    B = (dm.sh_degree + 1) ** 2
    f64 = lambda *shape: torch.empty((cap,) + shape, dtype=torch.float64, device=dev)
    buf = dict(rows=torch.empty(cap, dtype=torch.int64, device=dev), depth=f64(), mu2d=f64(2), sigma2d=f64(3),
               radius=f64(), window=torch.empty((cap, 4), dtype=torch.int32, device=dev), opacity=f64(),
               color=f64(3), color_pre=f64(3), shade_s=f64(), order=torch.empty(cap, dtype=torch.int64, device=dev))
    p = _lib.SSPrepared()
    for k, t in buf.items():
        setattr(p, k, t.data_ptr())
    p.capacity = cap
    vis = _lib.i64(0)
    camst, lst = camera_struct(pose, intr), light_struct(light_state)
    c.check(c.lib.ss_prepare_splats(c.handle, dm.struct(), camst, lst,
                                    render_opts((0, 0, 0), sub, extent_cutoff, 1), p, _lib.C.byref(vis)))
    M = int(vis.value)
    ext = dict(mu_cam=f64(3), J=f64(2, 3), sigma3d=f64(3, 3), cov_cam=f64(3, 3), view_dir=f64(3), view_dist=f64(),
               n_hat=f64(3), n_axis=torch.empty(cap, dtype=torch.int64, device=dev), Y=f64(B), albedo_est=f64(3),
               cos=f64(), vis=f64())
    e = _lib.SSPreparedExtras()
    for k, t in ext.items():
        setattr(e, k, t.data_ptr())
    c.check(c.lib.ss_prepare_extras(c.handle, dm.struct(), camst, lst, buf["rows"].data_ptr(), M, e))
    h = {k: t[:M].cpu().numpy() for k, t in buf.items()}
    x = {k: t[:M].cpu().numpy() for k, t in ext.items()}
    s = h["sigma2d"]
    Sig = np.stack([np.stack([s[:, 0], s[:, 1]], -1), np.stack([s[:, 1], s[:, 2]], -1)], -2)
    det = s[:, 0] * s[:, 2] - s[:, 1] * s[:, 1]
    inv = np.stack([np.stack([s[:, 2] / det, -s[:, 1] / det], -1), np.stack([-s[:, 1] / det, s[:, 0] / det], -1)], -2)
    R = pose.rotation() if hasattr(pose, "rotation") else quat_to_rotmat(pose.quaternion)
    inter = {"Y": x["Y"], "albedo_est": x["albedo_est"], "s": h["shade_s"], "cos": x["cos"], "vis": x["vis"]}
    return PreparedSplats(rows=h["rows"], mu_cam=x["mu_cam"], depth=h["depth"], mu2d=h["mu2d"], J=x["J"],
                          W=np.asarray(R, np.float64).T.copy(), Sigma3d=x["sigma3d"], cov_cam=x["cov_cam"],
                          Sigma2d=Sig, inv2d=inv, opacity=h["opacity"], color=h["color"], color_pre=h["color_pre"],
                          view_dir=x["view_dir"], view_dist=x["view_dist"], n_hat=x["n_hat"], n_axis=x["n_axis"],
                          shade_inter=inter, order=h["order"], radius=h["radius"],
                          windows=h["window"].astype(np.int64))


def splat_windows(mu2d, radius, width: int, height: int) -> np.ndarray:
    """(n, 4) int32 windows x0, x1, y0, y1 of ref render.py:293-301
    (splat_window), vectorised; an infinite radius covers the image."""
    mu2d = np.asarray(mu2d, np.float64).reshape(-1, 2)
    r = np.asarray(radius, np.float64).reshape(-1)
    big = 1 << 30
    fin = np.isfinite(r)
    rr = np.where(fin, r, 0.0)
    def lo(v):
        return np.clip(np.floor(v), -big, big).astype(np.int64)
    def hi(v):
        return np.clip(np.ceil(v), -big, big).astype(np.int64)
    x0 = np.maximum(lo(mu2d[:, 0] - rr), 0)
    x1 = np.minimum(hi(mu2d[:, 0] + rr) + 1, width)
    y0 = np.maximum(lo(mu2d[:, 1] - rr), 0)
    y1 = np.minimum(hi(mu2d[:, 1] + rr) + 1, height)
    w = np.stack([x0, x1, y0, y1], -1)
    w[~fin] = (0, width, 0, height)
    return w.astype(np.int32)


def composite(prep, intr, background, device=None):
    """ref render.py:317 -- front-to-back float64 composite of prepared
    splats on the GPU (ss_composite); returns (image (H, W, 3), T (H, W)) as
    host float64 arrays.  Uses prep.order, mu2d, radius, inv2d, opacity and
    color, exactly the fields the reference reads."""
    import torch
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    order = np.asarray(prep.order, np.int64)
    mu = np.asarray(prep.mu2d, np.float64)[order]
    inv = np.asarray(prep.inv2d, np.float64)[order]
    win = splat_windows(mu, np.asarray(prep.radius, np.float64)[order], intr.width, intr.height)
    t = lambda a, dt=torch.float64: torch.from_numpy(np.ascontiguousarray(a)).to(device=dev, dtype=dt)
    n = int(order.size)
    args = dict(mu=t(mu), inv=t(np.stack([inv[:, 0, 0], inv[:, 0, 1], inv[:, 1, 1]], -1) if n else np.zeros((0, 3))),
                op=t(np.asarray(prep.opacity, np.float64)[order]),
                col=t(np.asarray(prep.color, np.float64)[order]), win=t(win, torch.int32))
    H, W = intr.height, intr.width
    img = torch.empty((H, W, 3), dtype=torch.float64, device=dev)
    T = torch.empty((H, W), dtype=torch.float64, device=dev)
    c = _lib.ctx(dev.index)
    c.bind_stream()
    bg = (_lib.f64 * 3)(*[float(x) for x in np.asarray(background, np.float64).reshape(3)])
    p = (lambda k: args[k].data_ptr() if n else None)
    c.check(c.lib.ss_composite(c.handle, n, p("mu"), p("inv"), p("op"), p("col"), p("win"), W, H, bg,
                               img.data_ptr(), T.data_ptr()))
    return img.cpu().numpy(), T.cpu().numpy()


def tile_bins(model, pose, intr, index_subset=None, extent_cutoff=True):
    """Sort keys / tile ranges of K2-K4 for parity tests: returns
    (order_rows, ranges (T,2), pair_rank (P,))."""
    import torch
    dm, _ = as_device(model)
    c = _lib.ctx(dm.device.index)
    dev = dm.device
    sub = _subset_tensor(index_subset, dev)
    n = int(sub.numel()) if sub is not None else dm.count
    tiles = -(-intr.width // 16) * -(-intr.height // 16)
    o = render_opts((0, 0, 0), sub, extent_cutoff, 0)
    st = _lib.SSRenderStats()
    # first pass sizes the pair list
    c.check(c.lib.ss_debug_bins(c.handle, dm.struct(), camera_struct(pose, intr), o, None, max(n, 1), None, tiles,
                                None, 1 << 62, st))
    P = int(st.pairs)
    rows = torch.full((max(n, 1),), -1, dtype=torch.int64, device=dev)
    ranges = torch.zeros((tiles, 2), dtype=torch.int64, device=dev)
    ranks = torch.zeros(max(P, 1), dtype=torch.int64, device=dev)
    c.check(c.lib.ss_debug_bins(c.handle, dm.struct(), camera_struct(pose, intr), o, _lib.ptr(rows), max(n, 1),
                                _lib.ptr(ranges), tiles, _lib.ptr(ranks), max(P, 1), st))
    r = rows.cpu().numpy()[:n]
    return r[r >= 0], ranges.cpu().numpy(), ranks.cpu().numpy()[:P]


def update_light_visibility(model, depth_map, light_cam, bias: float = 0.02, changed=None) -> None:
    """ref render.py:350 -- writes model.light_visibility (replaced for host models).
    `changed`: optional device int32 tensor (zeroed by the caller) set to 1 when
    any bit flipped -- the server's packet test (ref server.py:406-409) on the device."""
    import torch
    dm, uploaded = as_device(model)
    if dm.count == 0:
        return
    c = _lib.ctx(dm.device.index)
    cam = _lib.SSOrthoCamera()
    cam.position = _lib.f64arr(light_cam.pose.position, 3)
    R = light_cam.pose.rotation() if hasattr(light_cam.pose, "rotation") else quat_to_rotmat(light_cam.pose.quaternion)
    cam.rot_cw = _lib.f64arr(np.asarray(R).ravel(), 9)
    cam.half_width, cam.half_height = float(light_cam.half_width), float(light_cam.half_height)
    cam.width, cam.height = int(light_cam.width), int(light_cam.height)
    depth = depth_map if isinstance(depth_map, torch.Tensor) else torch.from_numpy(
        np.ascontiguousarray(depth_map, np.float64))
    depth = depth.to(dm.device, torch.float64).contiguous()
    c.check(c.lib.ss_update_light_visibility_changed(c.handle, dm.struct(), _lib.ptr(depth), cam, float(bias),
                                                     _lib.ptr(changed)))
    if uploaded:
        model.light_visibility = dm.light_visibility.cpu().numpy().astype(np.float32)
