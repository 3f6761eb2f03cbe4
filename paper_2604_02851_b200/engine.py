"""Ray-cast scene engine on the GPU: the game-engine
stand-in that renders the optimiser's ground truth and the expansion inputs.

Drop-in for ref engine.py: `render_ground_truth` (engine.py:151),
`capture_input_buffers` (engine.py:161), `render_depth` (engine.py:192),
`render_ortho_depth` (engine.py:200) with the reference's signatures and host
numpy results, plus `render_ground_truth_device`, which leaves a float32
(H, W, 3) image in HBM for `optim.ReferenceView` (no host round trip in a
live loop).  One library call (`ss_engine_render`, one kernel) per image;
scenes are duck-typed (the reference's SceneDescription or
paper_2604_02851_b200.scene).  `build_dome_rig` / `build_light_camera` are
host camera-rig helpers (ref engine.py:208-246).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .geometry import CameraIntrinsics, OrthoCamera, look_at, quat_to_rotmat

GOLDEN_ANGLE = np.pi * (3.0 - np.sqrt(5.0))


@dataclass
class InputBuffers:
    """Per-pixel engine channels of one input camera (ref engine.py:36-51)."""

    pose: object
    intrinsics: object
    world_pos: np.ndarray
    valid: np.ndarray
    normal: np.ndarray
    albedo: np.ndarray
    shaded: np.ndarray
    object_id: np.ndarray
    depth: np.ndarray
    footprint: np.ndarray
    lit: np.ndarray


def _shape_kind(shape):
    if hasattr(shape, "radius"):
        return 1
    if hasattr(shape, "half_extents"):
        return 2
    if hasattr(shape, "normal"):
        return 0
    raise TypeError(f"unsupported shape {type(shape).__name__}")


def _tangents(shape):
    if hasattr(shape, "tangents"):
        return shape.tangents()
    n = np.asarray(shape.normal, np.float64)  # ref scene.py:41-46
    helper = np.array([1.0, 0, 0]) if abs(n[1]) > 0.9 else np.array([0, 1.0, 0])
    u = np.cross(helper, n)
    u = u / np.linalg.norm(u)
    return u, np.cross(n, u)


def scene_struct(scene, light=None, transforms=None):
    """(SSScene, keep-alive) for a scene; `transforms` {object_id: (q, t)}
    places dynamic objects (ref engine.py:81-84, 99-107)."""
    objs = scene.objects
    arr = (_lib.SSSceneObject * max(1, len(objs)))()
    for k, ob in enumerate(objs):
        s = arr[k]
        sh = ob.shape
        s.shape = _shape_kind(sh)
        s.object_id = int(ob.object_id)
        if s.shape == 0:
            s.a[:] = [float(x) for x in sh.point]
            s.b[:] = [float(x) for x in sh.normal]
            if sh.extent is not None:
                s.has_extent = 1
                s.extent[:] = [float(sh.extent[0]), float(sh.extent[1])]
                u, v = _tangents(sh)
                s.u[:] = [float(x) for x in u]
                s.v[:] = [float(x) for x in v]
        elif s.shape == 1:
            s.a[:] = [float(x) for x in sh.center]
            s.radius = float(sh.radius)
        else:
            s.a[:] = [float(x) for x in sh.center]
            s.b[:] = [float(x) for x in sh.half_extents]
        al = ob.albedo
        s.albedo_kind = 0 if al.kind == "solid" else 1
        s.color[:] = [float(x) for x in al.color]
        s.color2[:] = [float(x) for x in al.color2]
        s.scale = float(al.scale)
        if ob.object_id > 0 and transforms and ob.object_id in transforms:
            q, t = transforms[ob.object_id]
            s.has_transform = 1
            s.R[:] = [float(x) for x in np.asarray(quat_to_rotmat(q), np.float64).reshape(-1)]
            s.t[:] = [float(x) for x in np.asarray(t, np.float64)]
    lt = light if light is not None else scene.light
    sc = _lib.SSScene()
    sc.objects = C.cast(arr, C.POINTER(_lib.SSSceneObject))
    sc.n_objects = len(objs)
    sc.light_direction[:] = [float(x) for x in lt.direction]
    sc.light_intensity[:] = [float(x) for x in lt.intensity]
    sc.ambient[:] = [float(x) for x in lt.ambient]
    sc.background[:] = [float(x) for x in scene.background]
    return sc, arr


def _pinhole(pose, intr):
    cam = _lib.SSEngineCamera()
    cam.kind = 0
    cam.width, cam.height = int(intr.width), int(intr.height)
    cam.position[:] = [float(x) for x in np.asarray(pose.position, np.float64)]
    cam.R[:] = [float(x) for x in np.asarray(pose.rotation(), np.float64).reshape(-1)]
    cam.fx, cam.fy, cam.cx, cam.cy = float(intr.fx), float(intr.fy), float(intr.cx), float(intr.cy)
    cam.far = float(intr.far)
    cam.footprint_scale = float(2.0 * np.tan(intr.fov_y / 2.0) / intr.height)  # ref engine.py:167
    return cam


def _ortho(oc):
    cam = _lib.SSEngineCamera()
    cam.kind = 1
    cam.width, cam.height = int(oc.width), int(oc.height)
    cam.position[:] = [float(x) for x in np.asarray(oc.pose.position, np.float64)]
    cam.R[:] = [float(x) for x in np.asarray(oc.pose.rotation(), np.float64).reshape(-1)]
    cam.half_width, cam.half_height, cam.far = float(oc.half_width), float(oc.half_height), float(oc.far)
    return cam


@dataclass
class Hits:
    """Nearest hits of a ray batch (ref engine.py:24-33)."""

    t: np.ndarray             # ray parameter, inf where missed
    object_index: np.ndarray  # index into scene.objects, -1 where missed
    world_point: np.ndarray
    normal: np.ndarray        # world frame, unit, facing the ray origin
    albedo: np.ndarray

    @property
    def valid(self) -> np.ndarray:
        return np.isfinite(self.t)


def _broadcast_row(a):
    """The single (3,) vector a (..., 3) array repeats, or None."""
    flat = a.reshape(-1, 3) if a.flags.c_contiguous else None
    if flat is not None:
        return None
    st = a.strides[:-1]
    return a.reshape(-1)[:3].copy() if all(x == 0 for x in st) else None


def trace(scene, origins, dirs, transforms=None, device=None) -> Hits:
    """ref engine.py:88-127 on the GPU: nearest hit of every ray; `origins`
    broadcasts against `dirs`.  A `dirs` that is one broadcast vector (the
    shadow rays' -light.direction) follows numpy's broadcast-matmul order;
    anything else is taken row by row (numpy's BLAS order for >= 2 rays)."""
    import torch
    dev = _dev(device)
    dirs = np.asarray(dirs, dtype=np.float64)
    shape = dirs.shape[:-1]
    n = int(np.prod(shape)) if shape else 1
    out = {"t": torch.empty(max(n, 1), dtype=torch.float64, device=dev),
           "object_index": torch.empty(max(n, 1), dtype=torch.int32, device=dev),
           "world_pos": torch.empty((max(n, 1), 3), dtype=torch.float64, device=dev),
           "normal": torch.empty((max(n, 1), 3), dtype=torch.float64, device=dev),
           "albedo": torch.empty((max(n, 1), 3), dtype=torch.float64, device=dev)}
    if n:
        cam = _lib.SSEngineCamera()
        cam.kind, cam.width, cam.height = 2, n, 1
        drow = _broadcast_row(dirs)
        d_t = torch.from_numpy(drow if drow is not None else np.array(dirs, copy=True).reshape(-1, 3)).to(dev)
        o = np.asarray(origins, dtype=np.float64)
        orow = o.reshape(3) if o.shape == (3,) else _broadcast_row(np.broadcast_to(o, dirs.shape))
        o_t = torch.from_numpy(orow.copy() if orow is not None else
                               np.array(np.broadcast_to(o, dirs.shape), copy=True).reshape(-1, 3)).to(dev)
        cam.ray_origins, cam.ray_dirs = o_t.data_ptr(), d_t.data_ptr()
        cam.origin_stride = 0 if orow is not None else 3
        cam.dir_stride = 0 if drow is not None else 3
        _run(scene, cam, {"t": out["t"], "object_index": out["object_index"], "world_pos": out["world_pos"],
                          "normal": out["normal"], "albedo": out["albedo"]}, None, transforms, dev.index)
    h = {k: v[:n].cpu().numpy() for k, v in out.items()}
    # world_pos is written as 0 for misses; trace's world_point is origin + 0 * dir there
    t = h["t"].reshape(shape)
    ob = np.broadcast_to(np.asarray(origins, dtype=np.float64), dirs.shape)
    wp = np.where(np.isfinite(t)[..., None], h["world_pos"].reshape(dirs.shape), ob)
    return Hits(t=t, object_index=h["object_index"].reshape(shape).astype(np.int64), world_point=wp,
                normal=h["normal"].reshape(dirs.shape), albedo=h["albedo"].reshape(dirs.shape))


def light_occluded(scene, points, normals, light, transforms=None, device=None) -> np.ndarray:
    """ref engine.py:130-137: a shadow ray from p + 1e-5 n toward the light hits geometry."""
    points = np.asarray(points, dtype=np.float64)
    if points.size == 0:
        return np.zeros(points.shape[:-1], dtype=bool)
    origins = points + 1e-5 * np.asarray(normals, dtype=np.float64)
    d = np.broadcast_to(-np.asarray(light.direction, dtype=np.float64), points.shape)
    return trace(scene, origins, d, transforms, device).valid


def _run(scene, cam, bufs, light=None, transforms=None, device=None):
    c = _lib.ctx(device)
    c.bind_stream()
    sc, keep = scene_struct(scene, light, transforms)
    out = _lib.SSEngineOut()
    for k, t in bufs.items():
        setattr(out, k, t.data_ptr())
    c.check(c.lib.ss_engine_render(c.handle, C.byref(sc), C.byref(cam), C.byref(out)))
    del keep


def _dev(device):
    import torch
    return torch.device("cuda", torch.cuda.current_device() if device is None else device)


def render_ground_truth_device(scene, pose, intr, light=None, transforms=None, device=None, out=None):
    """(H, W, 3) float32 ground truth in HBM (ref engine.py:151-158, cast
    to float32 as the optimiser's views hold it).  `out` may be reused."""
    import torch
    dev = _dev(device)
    if out is None:
        out = torch.empty((intr.height, intr.width, 3), dtype=torch.float32, device=dev)
    _run(scene, _pinhole(pose, intr), {"gt_f32": out}, light, transforms, dev.index)
    return out


def render_ground_truth(scene, pose, intr, light=None, transforms=None, device=None) -> np.ndarray:
    """ref engine.py:151: (H, W, 3) float64, clipped to [0, 1]."""
    import torch
    dev = _dev(device)
    img = torch.empty((intr.height, intr.width, 3), dtype=torch.float64, device=dev)
    _run(scene, _pinhole(pose, intr), {"gt_f64": img}, light, transforms, dev.index)
    return img.cpu().numpy()


def capture_input_buffers(scene, pose, intr, light=None, transforms=None, device=None, as_tensors=False):
    """ref engine.py:161-189: every channel of one input camera (host numpy,
    or device tensors with `as_tensors`)."""
    import torch
    dev = _dev(device)
    H, W = intr.height, intr.width
    f64 = dict(dtype=torch.float64, device=dev)
    b = {"world_pos": torch.empty((H, W, 3), **f64), "valid": torch.empty((H, W), dtype=torch.uint8, device=dev),
         "normal": torch.empty((H, W, 3), **f64), "albedo": torch.empty((H, W, 3), **f64),
         "shaded": torch.empty((H, W, 3), **f64), "object_id": torch.empty((H, W), dtype=torch.int32, device=dev),
         "depth": torch.empty((H, W), **f64), "footprint": torch.empty((H, W), **f64),
         "lit": torch.empty((H, W), dtype=torch.uint8, device=dev)}
    _run(scene, _pinhole(pose, intr), b, light, transforms, dev.index)
    if as_tensors:
        b["valid"] = b["valid"].bool()
        b["lit"] = b["lit"].bool()
        return InputBuffers(pose=pose, intrinsics=intr, **b)
    h = {k: v.cpu().numpy() for k, v in b.items()}
    h["valid"] = h["valid"].astype(bool)
    h["lit"] = h["lit"].astype(bool)
    return InputBuffers(pose=pose, intrinsics=intr, **h)


def render_depth(scene, pose, intr, transforms=None, device=None, as_tensor=False):
    """ref engine.py:192-197: camera-space z per pixel, intr.far where no hit
    (host numpy, or the device tensor with `as_tensor`)."""
    import torch
    dev = _dev(device)
    d = torch.empty((intr.height, intr.width), dtype=torch.float64, device=dev)
    _run(scene, _pinhole(pose, intr), {"depth_or_far": d}, None, transforms, dev.index)
    return d if as_tensor else d.cpu().numpy()


def render_ortho_depth(scene, cam, transforms=None, device=None, as_tensor=False):
    """ref engine.py:200-205: distance along the projection direction, cam.far
    where no hit (host numpy, or the device tensor with `as_tensor`, e.g. for
    render.update_light_visibility)."""
    import torch
    dev = _dev(device)
    d = torch.empty((cam.height, cam.width), dtype=torch.float64, device=dev)
    _run(scene, _ortho(cam), {"depth_or_far": d}, None, transforms, dev.index)
    return d if as_tensor else d.cpu().numpy()


@dataclass
class SampleBatch:
    """Culled surface samples pooled across input cameras (ref engine.py:54-78)."""

    positions: object
    normals: object
    albedo: object
    object_ids: object
    footprints: object
    lit: object
    camera_indices: object

    @property
    def count(self) -> int:
        return int(self.positions.shape[0])


def _as_dev(a, dtype, dev):
    import torch
    if isinstance(a, torch.Tensor):
        return a.to(device=dev, dtype=dtype).contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a))).to(device=dev, dtype=dtype)


def cull_input_samples(buffers, device=None, as_tensors=False) -> SampleBatch:
    """ref engine.py:249-303 on the GPU: pool the valid samples of every input
    camera, voxel side 2 x the median footprint, per voxel only the samples of
    the least oblique camera (ties to the lower index).  `buffers` are
    InputBuffers with host (numpy) or device (torch) channels."""
    import torch
    dev = _dev(device)
    c = _lib.ctx(dev.index)
    c.bind_stream()
    cams = (_lib.SSCullCamera * max(1, len(buffers)))()
    keep = []
    total = 0
    for k, b in enumerate(buffers):
        ch = {"world_pos": _as_dev(b.world_pos, torch.float64, dev), "valid": _as_dev(b.valid, torch.uint8, dev),
              "normal": _as_dev(b.normal, torch.float64, dev), "albedo": _as_dev(b.albedo, torch.float64, dev),
              "object_id": _as_dev(b.object_id, torch.int32, dev), "footprint": _as_dev(b.footprint, torch.float64, dev),
              "lit": _as_dev(b.lit, torch.uint8, dev)}
        keep.append(ch)
        for name, t in ch.items():
            setattr(cams[k], name, t.data_ptr())
        cams[k].position[:] = [float(x) for x in np.asarray(b.pose.position, np.float64)]
        cams[k].pixels = int(ch["valid"].numel())
        total += cams[k].pixels
    cap = max(1, total)
    f64 = dict(dtype=torch.float64, device=dev)
    out = {"positions": torch.empty((cap, 3), **f64), "normals": torch.empty((cap, 3), **f64),
           "albedo": torch.empty((cap, 3), **f64), "object_ids": torch.empty(cap, dtype=torch.int32, device=dev),
           "footprints": torch.empty(cap, **f64), "lit": torch.empty(cap, dtype=torch.uint8, device=dev),
           "camera_indices": torch.empty(cap, dtype=torch.int32, device=dev)}
    sb = _lib.SSSampleBatch(*(out[k].data_ptr() for k in ("positions", "normals", "albedo", "object_ids", "footprints",
                                                          "lit", "camera_indices")))
    n = _lib.i64(0)
    side = _lib.f64(0.0)
    c.check(c.lib.ss_cull_input_samples(c.handle, cams, len(buffers), C.byref(sb), cap, C.byref(n), C.byref(side)))
    del keep
    n = int(n.value)
    res = {k: v[:n] for k, v in out.items()}
    res["lit"] = res["lit"].bool()
    if not as_tensors:
        res = {k: v.cpu().numpy() for k, v in res.items()}
    return SampleBatch(**res)


def init_gaussians(samples, sh_degree: int = 0, device=None, as_device: bool = False):
    """ref expansion.py:39-64 on the GPU: a batch of fresh Gaussians (one row
    per sample; isotropic scales log(max(footprint, 1e-6) / 2), identity
    rotation, opacity 0.5, SH DC reproducing the albedo).  Returns a host
    GaussianModel (all rows active), or a DeviceModel with `as_device`."""
    import torch
    from .model import DeviceModel
    dev = _dev(device)
    n = samples.count
    B = (sh_degree + 1) ** 2
    f32 = dict(dtype=torch.float32, device=dev)
    m = DeviceModel(torch.empty((n, 3), **f32), torch.empty((n, 3), **f32), torch.empty((n, 4), **f32),
                    torch.empty(n, **f32), torch.empty((n, 3, B), **f32), torch.empty(n, **f32),
                    torch.empty(n, dtype=torch.int32, device=dev), n, sh_degree)
    if n:
        c = _lib.ctx(dev.index)
        c.bind_stream()
        cols = {"positions": _as_dev(samples.positions, torch.float64, dev),
                "normals": _as_dev(samples.normals, torch.float64, dev),
                "albedo": _as_dev(samples.albedo, torch.float64, dev),
                "object_ids": _as_dev(samples.object_ids, torch.int32, dev),
                "footprints": _as_dev(samples.footprints, torch.float64, dev),
                "lit": _as_dev(samples.lit, torch.uint8, dev),
                "camera_indices": _as_dev(samples.camera_indices, torch.int32, dev)}
        sb = _lib.SSSampleBatch(*(cols[k].data_ptr() for k in ("positions", "normals", "albedo", "object_ids",
                                                                "footprints", "lit", "camera_indices")))
        st = m.struct()
        c.check(c.lib.ss_init_gaussians(c.handle, C.byref(sb), n, C.byref(st), 0))
        torch.cuda.current_stream(dev).synchronize()
        del cols
    return m if as_device else m.to_host()


def build_light_camera(aabb_lo, aabb_hi, direction, resolution: int = 256) -> OrthoCamera:
    """Orthographic camera along the light covering the AABB (ref engine.py:208-219)."""
    lo = np.asarray(aabb_lo, dtype=np.float64)
    hi = np.asarray(aabb_hi, dtype=np.float64)
    centre = (lo + hi) / 2
    r = float(np.linalg.norm(hi - lo) / 2) * 1.1 + 1e-3
    d = np.asarray(direction, dtype=np.float64)
    d = d / np.linalg.norm(d)
    eye = centre - d * (r + 1.0)
    return OrthoCamera(pose=look_at(eye, eye + d), half_width=r, half_height=r, width=resolution,
                       height=resolution, far=2 * r + 2.0)


def build_dome_rig(center, heading: float, n_cameras: int, radius: float, width: int = 64, height: int = 64,
                   fov_y: float = np.pi / 2, near: float = 0.05, far: float = 100.0):
    """Inward-looking cameras on the upper Fibonacci hemisphere (ref engine.py:222-246)."""
    if n_cameras < 1:
        raise ValueError("n_cameras must be >= 1")
    c = np.asarray(center, dtype=np.float64)
    poses = []
    for i in range(n_cameras):
        ct = 1.0 - i / n_cameras
        st = np.sqrt(max(0.0, 1.0 - ct * ct))
        phi = i * GOLDEN_ANGLE + heading
        poses.append(look_at(c + radius * np.array([st * np.cos(phi), ct, st * np.sin(phi)]), c))
    return poses, CameraIntrinsics(width=width, height=height, fov_y=fov_y, near=near, far=far)


__all__ = ["Hits", "trace", "light_occluded", "InputBuffers", "SampleBatch", "cull_input_samples", "init_gaussians", "scene_struct", "render_ground_truth", "render_ground_truth_device",
           "capture_input_buffers", "render_depth", "render_ortho_depth", "build_light_camera", "build_dome_rig"]
