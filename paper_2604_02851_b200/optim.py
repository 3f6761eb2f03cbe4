"""Optimize step on the B200 rasterizer: backward, Adam, view sharding.

Drop-in for ref pkg/src/splatstream/optim.py: ReferenceView (optim.py:34),
Gradients (optim.py:50), loss (optim.py:80), backward (optim.py:113),
LearningRates (optim.py:271), OptimizerState (optim.py:281), step
(optim.py:353).

Per view, ss_backward runs K1-K7 (preprocess, depth sort, binning, forward,
front-to-back backward with per-(tile, splat) partials, chain rule) and
accumulates into ONE flat float32 gradient buffer
[means | log_scales | quaternions | logit_opacities | sh_coeffs] over the
active rows.  With a process group the buffer and the loss are summed with a
single NCCL all-reduce (reference views sharded across GPUs,
SURVEY.md §8e); ss_adam_step then applies the batch-averaged Adam update
with float64 moments.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib, parallel
from .model import TRAINABLE, DeviceModel, as_device
from .render import _subset_tensor, camera_struct, light_struct, render_opts


@dataclass
class ReferenceView:
    pose: object
    intrinsics: object
    image: object                  # (H, W, 3) numpy (any float dtype) or torch float32 CUDA tensor
    light_state: object
    background: np.ndarray = field(default_factory=lambda: np.zeros(3))
    ready: bool = True

    def __post_init__(self):
        if tuple(self.image.shape[:2]) != (self.intrinsics.height, self.intrinsics.width):
            raise ValueError("reference image dimensions do not match intrinsics")


@dataclass
class Gradients:
    means: np.ndarray
    log_scales: np.ndarray
    quaternions: np.ndarray
    logit_opacities: np.ndarray
    sh_coeffs: np.ndarray

    def __iadd__(self, other):
        for k in TRAINABLE:
            setattr(self, k, getattr(self, k) + getattr(other, k))
        return self

    def scale(self, f: float):
        for k in TRAINABLE:
            setattr(self, k, getattr(self, k) * f)

    def per_gaussian_norm(self):
        return np.linalg.norm(self.means, axis=-1)


def loss(rendered, ground_truth) -> float:
    if rendered.shape != ground_truth.shape:
        raise ValueError(f"shape mismatch {rendered.shape} vs {ground_truth.shape}")
    return float(np.mean(np.abs(np.asarray(rendered, np.float64) - np.asarray(ground_truth, np.float64))))


def grad_layout(a: int, sh_degree: int):
    B = (sh_degree + 1) ** 2
    offs = [0, 3 * a, 6 * a, 10 * a, 11 * a, a * (11 + 3 * B)]
    shapes = [(a, 3), (a, 3), (a, 4), (a,), (a, 3, B)]
    return offs, shapes


def split_flat(flat, a, sh_degree):
    """Views of a flat gradient/moment buffer per parameter group."""
    offs, shapes = grad_layout(a, sh_degree)
    return {k: flat[offs[i]:offs[i + 1]].view(*shapes[i]) for i, k in enumerate(TRAINABLE)}


def _gt_tensor(view, device):
    import torch
    img = view.image
    if isinstance(img, torch.Tensor):
        t = img
        if t.device != device or t.dtype != torch.float32:
            t = t.to(device=device, dtype=torch.float32, non_blocking=True)
    else:
        t = torch.from_numpy(np.ascontiguousarray(img, np.float32)).to(device, non_blocking=True)
    return t.contiguous()


_COPY_STREAMS = {}
_GT_POOL = {}  # device index -> persistent ground-truth staging buffers


def _stage_ground_truth(views, device):
    """Device ground truth per view.  Host images (pinned CPU tensors or
    numpy) are all uploaded up front on a side stream, each view's kernels
    waiting only for its own copy, so H2D overlaps the previous views'
    backward passes."""
    import torch
    if all(isinstance(v.image, torch.Tensor) and v.image.is_cuda for v in views):
        return [_gt_tensor(v, device) for v in views]
    cur = torch.cuda.current_stream(device)
    cs = _COPY_STREAMS.get(device.index)
    if cs is None:
        cs = _COPY_STREAMS[device.index] = torch.cuda.Stream(device)
    # the copies wait for everything queued before this step, so one
    # persistent device buffer per view slot is safe to refill every step (no
    # allocator churn: fresh blocks would mean synchronising cudaMallocs)
    cs.wait_stream(cur)
    pool = _GT_POOL.setdefault(device.index, [])
    out = []
    with torch.cuda.stream(cs):
        for i, v in enumerate(views):
            img = v.image
            if not isinstance(img, torch.Tensor):
                img = torch.from_numpy(np.ascontiguousarray(img, np.float32))
            shape = tuple(img.shape)
            if i >= len(pool):
                pool.append(None)
            if pool[i] is None or tuple(pool[i].shape) != shape:
                pool[i] = torch.empty(shape, dtype=torch.float32, device=device)
            t = pool[i]
            t.copy_(img, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(cs)
            out.append((t, ev))
    return [_Pending(t, ev, cur) for t, ev in out]


class _Pending:
    """A device tensor whose producing copy must complete before use."""

    def __init__(self, t, ev, stream):
        self.t, self.ev, self.stream = t, ev, stream

    def wait(self):
        self.stream.wait_event(self.ev)
        return self.t


def _tile_hint(view, device):
    """Per-view device buffer of the last walk length of every tile (the
    library orders the next forward of this camera longest-first with it)."""
    import torch
    intr = view.intrinsics
    n = ((intr.width + 15) // 16) * ((intr.height + 15) // 16)
    h = view.__dict__.get("_tile_hint")
    if h is None or h.numel() != n or h.device != device:
        h = torch.full((n,), -1, dtype=torch.int32, device=device)  # 0xffffffff: unknown
        view.__dict__["_tile_hint"] = h
    return h


def _tile_order(view, device):
    """(per-view device buffer of the backward's tile walk order, valid?):
    the next forward of this camera reuses it instead of re-sorting."""
    import torch
    n = _tile_hint(view, device).numel()
    o = view.__dict__.get("_tile_order")
    if o is None or o.numel() != n or o.device != device:
        o = torch.zeros(n, dtype=torch.int32, device=device)
        view.__dict__["_tile_order"] = o
        view.__dict__["_tile_order_valid"] = False
    return o, view.__dict__.get("_tile_order_valid", False)


def backward_device(model: DeviceModel, view, grad_accum, loss_accum, index_subset=None, extent_cutoff=True,
                    precision=0, image_out=None, subset_tensor=None, gt=None, defer=None):
    """Accumulate one view's gradients into `grad_accum` (flat float32) and
    its loss into `loss_accum` (float64 CUDA scalar).  With `defer` =
    (g9, rinv) device buffers the view's screen-space gradients are left
    there for one `chain_views` call over all the step's views."""
    c = _lib.ctx(model.device.index)
    ready = None
    if gt is None:
        gt = _gt_tensor(view, model.device)
    elif isinstance(gt, _Pending):  # the library waits for the upload just before the backward blend
        ready = gt.ev.cuda_event
        gt = gt.t
    sub = subset_tensor if subset_tensor is not None else _subset_tensor(index_subset, model.device)
    st = _lib.SSRenderStats()
    c.check(c.lib.ss_backward(c.handle, model.struct(), camera_struct(view.pose, view.intrinsics),
                              light_struct(view.light_state),
                              render_opts(view.background, sub, extent_cutoff, precision, gt_ready=ready,
                                          tile_hint=_tile_hint(view, model.device), defer=defer,
                                          tile_order=_tile_order(view, model.device)),
                              _lib.ptr(gt), _lib.ptr(grad_accum), _lib.ptr(loss_accum), _lib.ptr(image_out), st))
    view.__dict__["_tile_order_valid"] = True
    return st


def backward(model, view: ReferenceView, index_subset=None, extent_cutoff: bool = True, precision: int = 0):
    """ref optim.py:113 -- (loss, Gradients over active rows, rendered image)."""
    import torch
    dm, _ = as_device(model)
    a = dm.active_count
    n = a * (11 + 3 * (dm.sh_degree + 1) ** 2)
    g = torch.zeros(max(n, 1), dtype=torch.float32, device=dm.device)
    L = torch.zeros(1, dtype=torch.float64, device=dm.device)
    H, W = view.intrinsics.height, view.intrinsics.width
    img = torch.empty((H, W, 3), dtype=torch.float64 if precision else torch.float32, device=dm.device)
    backward_device(dm, view, g, L, index_subset, extent_cutoff, precision, img)
    parts = split_flat(g[:n], a, dm.sh_degree)
    grads = Gradients(**{k: v.double().cpu().numpy() for k, v in parts.items()})
    return float(L.item()), grads, img.double().cpu().numpy()


@dataclass
class LearningRates:
    means: float = 2e-4
    log_scales: float = 5e-3
    quaternions: float = 1e-3
    logit_opacities: float = 5e-2
    sh_dc: float = 2.5e-3
    sh_rest: float = 1.25e-4


class OptimizerState:
    """Adam state for the active rows, HBM-resident (float64 moments).

    `.m[group]` / `.v[group]` are torch views into the flat moment buffers
    (same shapes as the reference's numpy arrays); `.age` (int64) and
    `.grad_ema` (float64) are torch tensors.  `step_count` is a host int.
    """

    GROUPS = TRAINABLE

    def __init__(self, model, lrs: Optional[LearningRates] = None, scene_extent: float = 1.0,
                 betas=(0.9, 0.999), eps: float = 1e-8, ema_beta: float = 0.99, device=None):
        import torch
        self.lrs = lrs or LearningRates()
        self.scene_extent = float(scene_extent)
        self.betas = tuple(betas)
        self.eps = float(eps)
        self.ema_beta = float(ema_beta)
        self.step_count = 0
        if device is None:
            device = model.device if isinstance(model, DeviceModel) else torch.device("cuda", torch.cuda.current_device())
        self.device = torch.device(device)
        self.sh_degree = int(model.sh_degree)
        self._alloc(int(model.active_count))

    def _alloc(self, a):
        import torch
        n = a * (11 + 3 * (self.sh_degree + 1) ** 2)
        self.m_flat = torch.zeros(max(n, 1), dtype=torch.float64, device=self.device)
        self.v_flat = torch.zeros(max(n, 1), dtype=torch.float64, device=self.device)
        self.age = torch.zeros(a, dtype=torch.int64, device=self.device)
        self.grad_ema = torch.zeros(a, dtype=torch.float64, device=self.device)

    @property
    def active_count(self) -> int:
        return int(self.age.shape[0])

    @property
    def m(self):
        return split_flat(self.m_flat, self.active_count, self.sh_degree)

    @property
    def v(self):
        return split_flat(self.v_flat, self.active_count, self.sh_degree)

    def hparams(self) -> _lib.SSAdamHparams:
        h = _lib.SSAdamHparams()
        h.lr_means = self.lrs.means * self.scene_extent
        h.lr_log_scales = self.lrs.log_scales
        h.lr_quaternions = self.lrs.quaternions
        h.lr_logit_opacities = self.lrs.logit_opacities
        h.lr_sh_dc = self.lrs.sh_dc
        h.lr_sh_rest = self.lrs.sh_rest
        h.beta1, h.beta2 = self.betas
        h.eps = self.eps
        h.ema_beta = self.ema_beta
        return h

    def resize(self, record):
        """Follow a model mutation record (ref optim.py:312-343)."""
        import torch
        kind = type(record).__name__
        a = self.active_count
        groups_m, groups_v = self.m, self.v
        if kind == "AppendRecord":
            if record.insert_at != a:
                raise ValueError("append record does not extend the active region")
            sel = None
            pad = int(record.count)
        elif kind == "PermuteRecord":
            sel = torch.as_tensor(np.asarray(record.permutation)[: record.new_active_count], device=self.device)
            if bool((sel >= a).any()):
                raise ValueError("permutation maps a frozen row into the active region")
            pad = 0
        elif kind == "PruneRecord":
            keep = np.ones(a, bool)
            idx = np.asarray(record.indices)
            keep[idx[idx < a]] = False
            sel = torch.as_tensor(np.flatnonzero(keep), device=self.device)
            pad = 0
        else:
            raise TypeError(f"unknown record {type(record)}")

        def remap(t):
            t = t if sel is None else t[sel]
            if pad:
                t = torch.cat([t, torch.zeros((pad,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)])
            return t

        new_m = {k: remap(v) for k, v in groups_m.items()}
        new_v = {k: remap(v) for k, v in groups_v.items()}
        age, ema = remap(self.age), remap(self.grad_ema)
        na = int(age.shape[0])
        self._alloc(na)
        for k in TRAINABLE:
            self.m[k].copy_(new_m[k])
            self.v[k].copy_(new_v[k])
        self.age.copy_(age)
        self.grad_ema.copy_(ema)


class StepWorkspace:
    """Reusable per-model device buffers for step() (gradient sum, loss, and
    the per-view screen-space gradients of the deferred chain rule)."""

    def __init__(self, model: DeviceModel):
        import torch
        a = model.active_count
        n = a * (11 + 3 * (model.sh_degree + 1) ** 2)
        self.n = n
        self.grad = torch.zeros(max(n, 1), dtype=torch.float32, device=model.device)
        self.loss = torch.zeros(1, dtype=torch.float64, device=model.device)
        self._defer = None

    def defer_buffers(self, views: int, n_in: int, device):
        """Per view: g9 (n_in, 9) float32 and rinv (n_in,) int32 device buffers
        (contiguous slices of one allocation, grown on demand)."""
        import torch
        d = self._defer
        if d is None or d[0].shape[0] < views or d[0].shape[1] < n_in:
            cap = max(n_in, 1, d[0].shape[1] if d is not None else 0)
            d = self._defer = (torch.empty((max(views, d[0].shape[0] if d is not None else 0), cap, 9),
                                           dtype=torch.float32, device=device),
                               torch.empty((max(views, d[0].shape[0] if d is not None else 0), cap), dtype=torch.int32,
                                           device=device))
        return [d[0][i, :n_in] for i in range(views)], [d[1][i, :n_in] for i in range(views)]


CHAIN_MAX_VIEWS = 16  # ss_chain_views


def chain_views(model: DeviceModel, views, g9, rinv, grad, subset_tensor=None):
    """The deferred chain rule of `views` (their backward_device calls got
    defer=(g9[i], rinv[i])): one pass over the rows, the gradient read and
    written once (ss_chain_views)."""
    import ctypes as C
    c = _lib.ctx(model.device.index)
    k = len(views)
    cams = (_lib.SSCamera * k)(*[camera_struct(v.pose, v.intrinsics) for v in views])
    lights = (_lib.SSLight * k)(*[light_struct(v.light_state) for v in views])
    gp = (C.c_void_p * k)(*[g9[i].data_ptr() for i in range(k)])
    rp = (C.c_void_p * k)(*[rinv[i].data_ptr() for i in range(k)])
    n_in = int(subset_tensor.numel()) if subset_tensor is not None else model.count
    c.check(c.lib.ss_chain_views(c.handle, model.struct(), cams, lights, k, gp, rp,
                                 _lib.ptr(subset_tensor) if subset_tensor is not None else None, n_in, _lib.ptr(grad)))


def step(model, state: OptimizerState, views, index_subset=None, extent_cutoff: bool = True, precision: int = 0,
         process_group=None, total_views: Optional[int] = None, workspace: Optional[StepWorkspace] = None,
         sync_loss: bool = True):
    """ref optim.py:353 -- one Adam step over the ready views; returns the mean loss.

    With `process_group`, `views` are this rank's shard; gradients and loss
    are all-reduced (sum) over the group and averaged over `total_views`
    (default: sum of the ranks' ready views).  `sync_loss=False` returns the
    device loss tensor instead of a host float (no host synchronisation).
    """
    import torch
    ready = [v for v in views if v.ready]
    if not ready and process_group is None:
        raise ValueError("no ready views")
    if state.active_count != model.active_count:
        raise ValueError("optimizer state out of sync with model")
    dm, uploaded = as_device(model)
    a = dm.active_count
    n_local = len(ready)
    if process_group is not None:
        total = int(total_views) if total_views is not None else \
            parallel.global_view_count(n_local, process_group, dm.device)
    else:
        total = n_local
    if total == 0:
        raise ValueError("no ready views")
    ws = workspace if workspace is not None else StepWorkspace(dm)
    ws.grad.zero_()
    ws.loss.zero_()
    sub = _subset_tensor(index_subset, dm.device)
    gts = _stage_ground_truth(ready, dm.device)
    n_in = int(sub.numel()) if sub is not None else dm.count
    if precision == 0 and a > 0 and n_in > 0:
        # chain rule of every view in one pass over the rows (ss_chain_views),
        # in batches of at most CHAIN_MAX_VIEWS views
        for b0 in range(0, len(ready), CHAIN_MAX_VIEWS):
            batch = list(zip(ready, gts))[b0:b0 + CHAIN_MAX_VIEWS]
            g9, rinv = ws.defer_buffers(len(batch), n_in, dm.device)
            for i, (v, gt) in enumerate(batch):
                backward_device(dm, v, ws.grad, ws.loss, None, extent_cutoff, precision, None, subset_tensor=sub,
                                gt=gt, defer=(g9[i], rinv[i]))
            chain_views(dm, [v for v, _ in batch], g9, rinv, ws.grad, sub)
    else:
        for v, gt in zip(ready, gts):
            backward_device(dm, v, ws.grad, ws.loss, None, extent_cutoff, precision, None, subset_tensor=sub, gt=gt)
    if process_group is not None:
        parallel.reduce_gradients(ws.grad, ws.loss, process_group)
    if a > 0:
        c = _lib.ctx(dm.device.index)
        st = _lib.SSAdamState()
        st.m = state.m_flat.data_ptr()
        st.v = state.v_flat.data_ptr()
        st.grad_ema = state.grad_ema.data_ptr()
        st.age = state.age.data_ptr()
        st.step_count = state.step_count
        c.check(c.lib.ss_adam_step(c.handle, dm.struct(), st, _lib.ptr(ws.grad), total, state.hparams()))
        state.step_count = int(st.step_count)
        if uploaded:
            dm.write_back(model, TRAINABLE, rows=a)
    if not sync_loss:
        return ws.loss / total
    return float(ws.loss.item()) / total
