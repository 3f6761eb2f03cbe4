"""ctypes binding of include/splatstream_b200.h (the C ABI).

The product has exactly one compute path: libsplat_b200.so on a CUDA device.
If the library is missing or no GPU is present, `lib()` raises -- there is no
CPU fallback.  Device buffers are torch CUDA tensors; only their data
pointers and sizes cross the boundary.
"""

from __future__ import annotations

import ctypes as C
import pathlib
import threading

import numpy as np

from .errors import ProtocolError

LIB_PATH = pathlib.Path(__file__).resolve().parent / "_lib" / "libsplat_b200.so"

SS_OK, SS_ERR_INVALID, SS_ERR_PROTOCOL, SS_ERR_CUDA, SS_ERR_CAPACITY = 0, -1, -2, -3, -4

vp = C.c_void_p
i32, i64, u64, f64 = C.c_int32, C.c_int64, C.c_uint64, C.c_double


class SSModel(C.Structure):
    _fields_ = [("means", vp), ("log_scales", vp), ("quaternions", vp), ("logit_opacities", vp),
                ("sh_coeffs", vp), ("light_visibility", vp), ("object_ids", vp),
                ("count", i32), ("active_count", i32), ("sh_degree", i32), ("param_dtype", i32)]


class SSCamera(C.Structure):
    _fields_ = [("position", f64 * 3), ("rot_cw", f64 * 9), ("fx", f64), ("fy", f64), ("cx", f64),
                ("cy", f64), ("near_plane", f64), ("width", i32), ("height", i32)]


class SSLight(C.Structure):
    _fields_ = [("direction", f64 * 3), ("intensity", f64 * 3), ("ambient_bands", i32), ("_pad", i32),
                ("ambient", f64 * 48)]


class SSRenderOpts(C.Structure):
    _fields_ = [("background", f64 * 3), ("subset", vp), ("subset_count", i32), ("extent_cutoff", i32),
                ("precision", i32), ("deterministic", i32), ("gt_ready", vp), ("tile_hint", vp),
                ("tile_hint_len", i64), ("defer_g9", vp), ("defer_rinv", vp), ("tile_order", vp),
                ("tile_order_valid", i32), ("_pad2", i32), ("bins_status", vp)]


class SSRenderStats(C.Structure):
    _fields_ = [("visible", i64), ("pairs", i64), ("tiles", i64)]


class SSAdamHparams(C.Structure):
    _fields_ = [("lr_means", f64), ("lr_log_scales", f64), ("lr_quaternions", f64),
                ("lr_logit_opacities", f64), ("lr_sh_dc", f64), ("lr_sh_rest", f64),
                ("beta1", f64), ("beta2", f64), ("eps", f64), ("ema_beta", f64)]


class SSAdamState(C.Structure):
    _fields_ = [("m", vp), ("v", vp), ("grad_ema", vp), ("age", vp), ("step_count", i32), ("skip_if", vp)]


class SSPrepared(C.Structure):
    _fields_ = [("rows", vp), ("depth", vp), ("mu2d", vp), ("sigma2d", vp), ("radius", vp), ("window", vp),
                ("opacity", vp), ("color", vp), ("color_pre", vp), ("shade_s", vp), ("order", vp),
                ("capacity", i64)]


class SSPreparedExtras(C.Structure):
    _fields_ = [(k, vp) for k in ("mu_cam", "J", "sigma3d", "cov_cam", "view_dir", "view_dist", "n_hat", "n_axis", "Y",
                                  "albedo_est", "cos", "vis")]


class SSDeltaJob(C.Structure):
    _fields_ = [("attribute_id", i32), ("in_dtype", i32), ("cur", vp), ("base", vp), ("new_base", vp),
                ("rows", i64), ("dims", i32), ("inner", i32), ("row_stride", i64), ("outer", i32), ("col0", i32),
                ("gating_threshold", f64), ("out", vp), ("out_cap", u64), ("out_len", vp)]


class SSIngestStatus(C.Structure):
    _fields_ = [("code", i32), ("_pad", i32), ("offset", i64)]


class SSDeltaApply(C.Structure):
    _fields_ = [("attribute_id", i32), ("mode", i32), ("dims", i32), ("bits", i32), ("count", i64), ("k", i64),
                ("lo", f64), ("hi", f64), ("block", vp), ("block_len", i64), ("baseline", vp), ("target", vp),
                ("row_stride", i64), ("inner", i32), ("outer", i32), ("col0", i32), ("_pad", i32), ("status", vp)]


class SSSnapshotDecode(C.Structure):
    _fields_ = [("model", SSModel), ("profile_id", i32), ("_pad", i32), ("aabb_lo", f64 * 3), ("aabb_hi", f64 * 3),
                ("block", vp), ("block_len", i64), ("status", vp)]


class SSPoolCamera(C.Structure):
    _fields_ = [("position", f64 * 3), ("rot_cw", f64 * 9), ("fx", f64), ("fy", f64), ("cx", f64), ("cy", f64),
                ("near_plane", f64), ("far_plane", f64), ("tx", f64), ("ty", f64), ("nx", f64), ("ny", f64),
                ("width", i32), ("height", i32), ("depth", vp)]


class SSSelect(C.Structure):
    _fields_ = [("kind", i32), ("n_cameras", i32), ("n", i64), ("age", vp), ("grad_ema", vp),
                ("age_threshold", i64), ("grad_threshold", f64), ("logits", vp), ("opacity_floor", f64),
                ("cells", vp), ("origin", f64 * 3), ("cell_size", f64), ("margin", f64),
                ("cameras", C.POINTER(SSPoolCamera)), ("row_ids", vp)]


class SSGridSpec(C.Structure):
    _fields_ = [("origin", f64 * 3), ("cell_size", f64)]


class SSSceneObject(C.Structure):
    _fields_ = [("shape", i32), ("object_id", i32), ("albedo_kind", i32), ("has_extent", i32), ("has_transform", i32),
                ("_pad", i32), ("a", f64 * 3), ("b", f64 * 3), ("radius", f64), ("extent", f64 * 2), ("u", f64 * 3),
                ("v", f64 * 3), ("color", f64 * 3), ("color2", f64 * 3), ("scale", f64), ("R", f64 * 9), ("t", f64 * 3)]


class SSScene(C.Structure):
    _fields_ = [("objects", C.POINTER(SSSceneObject)), ("n_objects", i32), ("_pad", i32), ("light_direction", f64 * 3),
                ("light_intensity", f64 * 3), ("ambient", f64 * 3), ("background", f64 * 3)]


class SSEngineCamera(C.Structure):
    _fields_ = [("kind", i32), ("width", i32), ("height", i32), ("_pad", i32), ("position", f64 * 3), ("R", f64 * 9),
                ("fx", f64), ("fy", f64), ("cx", f64), ("cy", f64), ("half_width", f64), ("half_height", f64),
                ("far", f64), ("footprint_scale", f64), ("ray_origins", vp), ("ray_dirs", vp), ("origin_stride", i32),
                ("dir_stride", i32)]


class SSEngineOut(C.Structure):
    _fields_ = [(n, vp) for n in ("gt_f32", "gt_f64", "depth_or_far", "world_pos", "valid", "normal", "albedo",
                                  "shaded", "object_id", "depth", "footprint", "lit", "t", "object_index")]


class SSCullCamera(C.Structure):
    _fields_ = [(n, vp) for n in ("world_pos", "valid", "normal", "albedo", "object_id", "footprint", "lit")] + \
               [("position", f64 * 3), ("pixels", i64)]


class SSSampleBatch(C.Structure):
    _fields_ = [(n, vp) for n in ("positions", "normals", "albedo", "object_ids", "footprints", "lit",
                                  "camera_indices")]


class SSOrthoCamera(C.Structure):
    _fields_ = [("position", f64 * 3), ("rot_cw", f64 * 9), ("half_width", f64), ("half_height", f64),
                ("width", i32), ("height", i32)]


_SIGS = {
    "ss_abi_version": (i32, []),
    "ss_ctx_create": (i32, [i32, C.POINTER(vp)]),
    "ss_ctx_destroy": (None, [vp]),
    "ss_last_error": (C.c_char_p, [vp]),
    "ss_set_stream": (i32, [vp, vp]),
    "ss_pair_capacity": (i64, [vp, i64]),
    "ss_host_syncs": (i64, [vp]),
    "ss_grad_layout": (i64, [i64, i32, C.POINTER(i64)]),
    "ss_set_timing": (i32, [vp, i32]),
    "ss_get_timing": (i32, [vp, C.POINTER(f64), C.POINTER(i64), C.POINTER(u64), i32]),
    "ss_measure_fp32_peak": (i32, [vp, C.POINTER(f64)]),
    "ss_render": (i32, [vp, C.POINTER(SSModel), C.POINTER(SSCamera), C.POINTER(SSLight),
                        C.POINTER(SSRenderOpts), vp, vp, C.POINTER(SSRenderStats)]),
    "ss_prepare_splats": (i32, [vp, C.POINTER(SSModel), C.POINTER(SSCamera), C.POINTER(SSLight),
                                C.POINTER(SSRenderOpts), C.POINTER(SSPrepared), C.POINTER(i64)]),
    "ss_debug_bins": (i32, [vp, C.POINTER(SSModel), C.POINTER(SSCamera), C.POINTER(SSRenderOpts), vp, i64, vp,
                            i64, vp, i64, C.POINTER(SSRenderStats)]),
    "ss_backward": (i32, [vp, C.POINTER(SSModel), C.POINTER(SSCamera), C.POINTER(SSLight),
                          C.POINTER(SSRenderOpts), vp, vp, vp, vp, C.POINTER(SSRenderStats)]),
    "ss_adam_step": (i32, [vp, C.POINTER(SSModel), C.POINTER(SSAdamState), vp, i32, C.POINTER(SSAdamHparams)]),
    "ss_encode_delta": (i32, [vp, i32, vp, i32, vp, vp, i64, i32, f64, vp, u64, vp]),
    "ss_delta_bound": (u64, [i32, i64, i32]),
    "ss_encode_delta_batch": (i32, [vp, C.POINTER(SSDeltaJob), i32]),
    "ss_encode_snapshot": (i32, [vp, C.POINTER(SSModel), i32, vp, u64, vp, vp, vp]),
    "ss_snapshot_bound": (u64, [i64, i32, i32]),
    "ss_encode_light_visibility": (i32, [vp, vp, i64, vp, u64, vp]),
    "ss_host_zlib_compress": (i32, [vp, u64, vp, u64, C.POINTER(u64)]),
    "ss_host_zlib_bound": (u64, [u64]),
    "ss_crc32": (i32, [vp, vp, vp, u64, vp]),
    "ss_crc32_combine": (C.c_uint32, [C.c_uint32, C.c_uint32, u64]),
    "ss_update_light_visibility": (i32, [vp, C.POINTER(SSModel), vp, C.POINTER(SSOrthoCamera), f64]),
    "ss_update_light_visibility_changed": (i32, [vp, C.POINTER(SSModel), vp, C.POINTER(SSOrthoCamera), f64, vp]),
    "ss_apply_object_transform": (i32, [vp, C.POINTER(SSModel), i32, vp, vp, C.POINTER(f64), C.POINTER(f64)]),
    "ss_refresh_object_locals": (i32, [vp, C.POINTER(SSModel), i32, i32, vp, vp, C.POINTER(f64),
                                       C.POINTER(f64)]),
    "ss_refresh_object_locals_rows": (i32, [vp, C.POINTER(SSModel), i32, vp, i64, vp, vp, C.POINTER(f64),
                                            C.POINTER(f64)]),
    "ss_decode_delta": (i32, [vp, C.POINTER(SSDeltaApply), vp, vp]),
    "ss_apply_delta": (i32, [vp, C.POINTER(SSDeltaApply), vp]),
    "ss_decode_snapshot": (i32, [vp, C.POINTER(SSSnapshotDecode)]),
    "ss_select_rows": (i32, [vp, C.POINTER(SSSelect), vp, C.POINTER(i64)]),
    "ss_gather_rows": (i32, [vp, C.POINTER(SSModel), C.POINTER(SSModel), vp, i64, C.POINTER(SSModel)]),
    "ss_cull_input_samples": (i32, [vp, C.POINTER(SSCullCamera), i32, C.POINTER(SSSampleBatch), i64, C.POINTER(i64),
                                    C.POINTER(f64)]),
    "ss_init_gaussians": (i32, [vp, C.POINTER(SSSampleBatch), i64, C.POINTER(SSModel), i64]),
    "ss_composite": (i32, [vp, i64, vp, vp, vp, vp, vp, i32, i32, C.POINTER(f64), vp, vp]),
    "ss_chain_views": (i32, [vp, C.POINTER(SSModel), vp, vp, i32, C.POINTER(vp), C.POINTER(vp), vp, i64, vp]),
    "ss_chain_views_range": (i32, [vp, C.POINTER(SSModel), vp, vp, i32, C.POINTER(vp), C.POINTER(vp), vp, i64, i64,
                                   i64, i64, vp, i64]),
    "ss_chain_views_range_init": (i32, [vp, C.POINTER(SSModel), vp, vp, i32, C.POINTER(vp), C.POINTER(vp), vp, i64,
                                        i64, i64, i64, vp, i64, i32]),
    "ss_sum_f64": (i32, [vp, vp, i64, vp]),
    "ss_debug_bwd_stats": (i32, [vp, C.POINTER(u64), i32]),
    "ss_prepare_extras": (i32, [vp, C.POINTER(SSModel), C.POINTER(SSCamera), C.POINTER(SSLight), vp, i64,
                                C.POINTER(SSPreparedExtras)]),
    "ss_adam_step_ld": (i32, [vp, C.POINTER(SSModel), C.POINTER(SSAdamState), vp, i64, i32,
                              C.POINTER(SSAdamHparams)]),
    "ss_adam_step_peers": (i32, [vp, C.POINTER(SSModel), C.POINTER(SSAdamState), vp, i64, i32,
                                 C.POINTER(SSAdamHparams), i32, C.POINTER(vp)]),
    "ss_engine_render": (i32, [vp, C.POINTER(SSScene), C.POINTER(SSEngineCamera), C.POINTER(SSEngineOut)]),
    "ss_grid_rebuild": (i32, [vp, vp, i64, C.POINTER(SSGridSpec), vp, vp, vp, vp, C.POINTER(i64)]),
    "ss_zigzag_varints": (i32, [vp, vp, i64, vp, u64, C.POINTER(u64)]),
}

_lib = None
_lock = threading.Lock()


def load_library(path=LIB_PATH):
    """Load and type the shared library (works without a GPU)."""
    global _lib
    with _lock:
        if _lib is None:
            if not pathlib.Path(path).exists():
                raise RuntimeError(
                    f"{path} is missing: build it with `python -m paper_2604_02851_b200._build` "
                    "(there is no CPU fallback)")
            lib = C.CDLL(str(path))
            for name, (res, args) in _SIGS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


class Context:
    """One ss_ctx per (device, thread); binds the current torch stream per call."""

    def __init__(self, device: int):
        self.lib = load_library()
        h = vp()
        rc = self.lib.ss_ctx_create(device, C.byref(h))
        if rc != SS_OK:
            raise RuntimeError(f"ss_ctx_create failed ({rc}) on cuda:{device}")
        self.handle = h
        self.device = device

    def check(self, rc: int):
        if rc == SS_OK:
            return
        msg = self.lib.ss_last_error(self.handle).decode(errors="replace")
        if rc == SS_ERR_INVALID:
            raise ValueError(msg)
        if rc == SS_ERR_PROTOCOL:
            raise ProtocolError(msg)
        raise RuntimeError(f"splatstream_b200 error {rc}: {msg}")

    def bind_stream(self):
        import torch
        s = torch.cuda.current_stream(self.device)
        self.check(self.lib.ss_set_stream(self.handle, vp(s.cuda_stream)))

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                self.lib.ss_ctx_destroy(self.handle)
        except Exception:
            pass


_ctx = threading.local()


def ctx(device=None) -> Context:
    """The calling thread's context for `device` (default: current CUDA device)."""
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("splatstream_b200 needs a CUDA device (there is no CPU fallback)")
    dev = torch.cuda.current_device() if device is None else int(device)
    cache = getattr(_ctx, "by_dev", None)
    if cache is None:
        cache = _ctx.by_dev = {}
    if dev not in cache:
        cache[dev] = Context(dev)
    c = cache[dev]
    c.bind_stream()
    return c


def lane_ctx(device: int, lane: int) -> Context:
    """Context of view lane `lane` on `device` (lane 0 is ctx(device)); each
    lane owns its own scratch arena, so lanes bound to different streams run
    concurrently.  Binds the current torch stream."""
    if lane == 0:
        return ctx(device)
    cache = getattr(_ctx, "lanes", None)
    if cache is None:
        cache = _ctx.lanes = {}
    key = (int(device), int(lane))
    c = cache.get(key)
    if c is None:
        c = cache[key] = Context(int(device))
        main = ctx(device)
        cap = c.lib.ss_pair_capacity(main.handle, 0)
        if cap > 0:
            c.lib.ss_pair_capacity(c.handle, cap)
        if getattr(main, "timing", False):
            c.check(c.lib.ss_set_timing(c.handle, 1))
            c.timing = True
    c.bind_stream()
    return c


_LANE_STREAMS = {}


def lane_stream(device: int, lane: int):
    """The torch stream of view lane `lane` >= 1 on `device` (created once;
    lane 0 is the caller's current stream)."""
    import torch
    key = (int(device), int(lane))
    s = _LANE_STREAMS.get(key)
    if s is None:
        s = _LANE_STREAMS[key] = torch.cuda.Stream(torch.device("cuda", int(device)))
    return s


def device_contexts(device: int):
    """Every context of `device` in this thread (the main one first)."""
    out = [ctx(device)]
    for (d, _), c in sorted(getattr(_ctx, "lanes", {}).items()):
        if d == int(device):
            out.append(c)
    return out


def pair_capacity(device: int, cap: int = 0) -> int:
    """ss_pair_capacity on every context of the device; returns the main one's."""
    cs = device_contexts(device)
    for c in cs[1:]:
        c.lib.ss_pair_capacity(c.handle, cap)
    return cs[0].lib.ss_pair_capacity(cs[0].handle, cap)


def host_syncs(device: int) -> int:
    """ss_host_syncs summed over the device's contexts."""
    return sum(c.lib.ss_host_syncs(c.handle) for c in device_contexts(device))


KERNEL_CLASSES = ("preprocess", "depth_sort", "binning", "tile_sort", "blend_forward", "blend_backward",
                  "chain_rule", "adam", "encoders")


def set_timing(c: "Context", on: bool):
    """Per-kernel-class timing on c and on every view lane of its device."""
    for x in device_contexts(c.device):
        x.check(x.lib.ss_set_timing(x.handle, 1 if on else 0))
        x.timing = bool(on)


def get_timing(c: "Context", reset=True):
    """{class: (ms, launch groups)}, counters (evaluated pairs, kernel launches),
    summed over c's device's contexts (view lanes overlap in time: the sum
    is device time per class, not wall time)."""
    tot = {k: [0.0, 0] for k in KERNEL_CLASSES}
    cnt_tot = [0, 0, 0, 0]
    for x in device_contexts(c.device):
        ms = (f64 * 9)()
        groups = (i64 * 9)()
        cnt = (u64 * 4)()
        x.check(x.lib.ss_get_timing(x.handle, ms, groups, cnt, 1 if reset else 0))
        for i, k in enumerate(KERNEL_CLASSES):
            tot[k][0] += ms[i]
            tot[k][1] += groups[i]
        cnt_tot = [a + b for a, b in zip(cnt_tot, cnt)]
    return {k: (v[0], v[1]) for k, v in tot.items()}, cnt_tot


def ptr(t) -> vp:
    """Device pointer of a torch tensor (None -> NULL)."""
    return vp(0) if t is None else vp(t.data_ptr())


def f64arr(values, n):
    a = (f64 * n)()
    v = np.asarray(values, np.float64).ravel()
    for i in range(min(n, v.size)):
        a[i] = float(v[i])
    return a
