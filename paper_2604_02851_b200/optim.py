"""Optimize step on the B200 rasterizer: backward, Adam, view sharding.

Drop-in for ref pkg/src/splatstream/optim.py: ReferenceView (optim.py:34),
Gradients (optim.py:50), loss (optim.py:80), backward (optim.py:113),
LearningRates (optim.py:271), OptimizerState (optim.py:281), step
(optim.py:353).

Per view, ss_backward runs K1-K6 (preprocess, depth sort, binning, forward,
front-to-back backward with per-(tile, splat) partials) and the fixed-order
partial sums, leaving per-row screen-space gradients; ONE chain-rule pass
over the rows (ss_chain_views_range) turns every view's records into the
flat float32 gradient [means | log_scales | quaternions | logit_opacities |
sh_coeffs], and ss_adam_step applies the batch-averaged Adam update with
float64 moments.  On N GPUs the same step is sharded by views and rows with
an exchange of the screen-space records (parallel.py); its result is
bit-identical to the single-GPU step.
"""

from __future__ import annotations

import os
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
    backward passes.  Two persistent buffer sets alternate between calls:
    a step's uploads wait only for the step before the previous one (the
    last reader of their set), so they run during the previous step instead
    of stalling the start of this one."""
    import torch
    if all(isinstance(v.image, torch.Tensor) and v.image.is_cuda for v in views):
        return [_gt_tensor(v, device) for v in views]
    cur = torch.cuda.current_stream(device)
    cs = _COPY_STREAMS.get(device.index)
    if cs is None:
        cs = _COPY_STREAMS[device.index] = torch.cuda.Stream(device)
    st = _GT_POOL.setdefault(device.index, {"sets": ([], []), "k": 0, "prev": None})
    k = st["k"]
    st["k"] = k + 1
    pool = st["sets"][k % 2]
    # everything queued so far (through the previous step); the set used two
    # calls ago was last read before the event recorded at the previous call
    now = torch.cuda.Event()
    now.record(cur)
    if st["prev"] is not None:
        cs.wait_event(st["prev"])
    else:
        cs.wait_stream(cur)
    st["prev"] = now
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
                if pool[i] is not None:  # a reshaped slot: the old buffer may still be read
                    cs.wait_stream(cur)
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
                    precision=0, image_out=None, subset_tensor=None, gt=None, defer=None, deterministic=True,
                    bins_status=None, ctx=None):
    """Accumulate one view's gradients into `grad_accum` (flat float32) and
    its loss into `loss_accum` (float64 CUDA scalar).  With `defer` =
    (g9, rinv) device buffers the view's screen-space gradients are left
    there for one `chain_views` call over all the step's views.  `ctx`: the
    library context to run on (a view lane's, see _DeviceKernels)."""
    c = ctx if ctx is not None else _lib.ctx(model.device.index)
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
                              render_opts(view.background, sub, extent_cutoff, precision, int(bool(deterministic)),
                                          gt_ready=ready,
                                          tile_hint=_tile_hint(view, model.device), defer=defer,
                                          tile_order=_tile_order(view, model.device), bins_status=bins_status),
                              _lib.ptr(gt), _lib.ptr(grad_accum), _lib.ptr(loss_accum), _lib.ptr(image_out), st))
    view.__dict__["_tile_order_valid"] = True
    return st


def backward(model, view: ReferenceView, index_subset=None, extent_cutoff: bool = True, precision: int = 0,
             deterministic: bool = True):
    """ref optim.py:113 -- (loss, Gradients over active rows, rendered image).
    deterministic=False: the throughput mode (float atomics, see ss_render_opts)."""
    import torch
    dm, _ = as_device(model, keep_f64=precision == 1)
    a = dm.active_count
    n = a * (11 + 3 * (dm.sh_degree + 1) ** 2)
    g = torch.zeros(max(n, 1), dtype=torch.float32, device=dm.device)
    L = torch.zeros(1, dtype=torch.float64, device=dm.device)
    H, W = view.intrinsics.height, view.intrinsics.width
    img = torch.empty((H, W, 3), dtype=torch.float64 if precision else torch.float32, device=dm.device)
    backward_device(dm, view, g, L, index_subset, extent_cutoff, precision, img, deterministic=deterministic)
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
    """Adam state for the active rows, HBM-resident (float64 moments, int64
    age, float64 grad-norm EMA).

    Reference view (ref optim.py:281-310): `.m[group]`, `.v[group]`, `.age`,
    `.grad_ema` are numpy arrays with the reference's shapes; they are host
    mirrors of the device buffers, taken when first read after a device
    update, and anything written into them is uploaded before the next device
    use (step, resize, pool policies) -- the reference's tests read and write
    them directly (pkg/tests/test_optim.py:342-376).  `step_count` is a host int.

    With `process_group` (the view-sharded step, parallel.py) each rank holds
    only its row shard of the moments/age/EMA (ZeRO-1); the numpy views are
    then the shard's, and `device_stats()` gathers the full age/EMA.
    """

    GROUPS = TRAINABLE

    def __init__(self, model, lrs: Optional[LearningRates] = None, scene_extent: float = 1.0,
                 betas=(0.9, 0.999), eps: float = 1e-8, ema_beta: float = 0.99, device=None, process_group=None):
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
        self.process_group = process_group
        if process_group is not None:
            import torch.distributed as dist
            self._world, self._rank = dist.get_world_size(process_group), dist.get_rank(process_group)
        else:
            self._world, self._rank = 1, 0
        self._host = None
        self._dirty = False
        self._alloc(int(model.active_count))

    # ---- layout
    @property
    def plan(self) -> parallel.ShardPlan:
        return parallel.ShardPlan(self._world, self._rank, self._active)

    @property
    def ld(self) -> int:
        """Rows per group of this rank's moment / gradient layout."""
        return self._active if self._world == 1 else self.plan.R

    def _alloc(self, a):
        import torch
        self._active = int(a)
        ld = self.ld
        n = ld * (11 + 3 * (self.sh_degree + 1) ** 2)
        self.m_dev = torch.zeros(max(n, 1), dtype=torch.float64, device=self.device)
        self.v_dev = torch.zeros(max(n, 1), dtype=torch.float64, device=self.device)
        self.age_dev = torch.zeros(max(ld, 1), dtype=torch.int64, device=self.device)
        self.ema_dev = torch.zeros(max(ld, 1), dtype=torch.float64, device=self.device)
        self._host = None
        self._dirty = False

    @property
    def active_count(self) -> int:
        return self._active

    def _groups(self, flat):
        """Per-group views of a flat moment buffer (this rank's rows)."""
        ld, rows = self.ld, (self._active if self._world == 1 else self.plan.rows)
        parts = split_flat(flat, ld, self.sh_degree) if ld > 0 else split_flat(flat[:0], 0, self.sh_degree)
        return {k: v[:rows] for k, v in parts.items()}

    # ---- reference-visible numpy mirror (write-back)
    def _mirror(self):
        if self._host is None:
            rows = self._active if self._world == 1 else self.plan.rows
            self._host = dict(m={k: v.cpu().numpy() for k, v in self._groups(self.m_dev).items()},
                              v={k: v.cpu().numpy() for k, v in self._groups(self.v_dev).items()},
                              age=self.age_dev[:rows].cpu().numpy(), grad_ema=self.ema_dev[:rows].cpu().numpy())
        self._dirty = True  # handed out: the caller may write into it
        return self._host

    def sync_device(self):
        """Upload host-mirror writes (before any device use of the state)."""
        import torch
        if self._host is not None and self._dirty:
            h = self._host
            for key, flat in (("m", self.m_dev), ("v", self.v_dev)):
                for k, t in self._groups(flat).items():
                    t.copy_(torch.from_numpy(np.ascontiguousarray(h[key][k], np.float64)).reshape(t.shape))
            rows = len(h["age"])
            self.age_dev[:rows].copy_(torch.from_numpy(np.ascontiguousarray(h["age"], np.int64)))
            self.ema_dev[:rows].copy_(torch.from_numpy(np.ascontiguousarray(h["grad_ema"], np.float64)))
        self._host = None
        self._dirty = False

    @property
    def m(self):
        return self._mirror()["m"]

    @property
    def v(self):
        return self._mirror()["v"]

    @property
    def age(self):
        return self._mirror()["age"]

    @age.setter
    def age(self, value):
        self._mirror()["age"][...] = value

    @property
    def grad_ema(self):
        return self._mirror()["grad_ema"]

    @grad_ema.setter
    def grad_ema(self, value):
        self._mirror()["grad_ema"][...] = value

    # ---- device views
    def device_groups(self):
        """(m, v) per-group device views of this rank's rows."""
        self.sync_device()
        return self._groups(self.m_dev), self._groups(self.v_dev)

    def device_stats(self):
        """(age, grad_ema) device tensors over ALL active rows (gathered from
        the ranks' shards in the sharded step) for the pool policies."""
        import torch
        self.sync_device()
        a = self._active
        if self._world == 1:
            return self.age_dev[:a], self.ema_dev[:a]
        coll = parallel.Collectives(self.process_group)
        R = self.plan.R
        age = torch.empty(self._world * R, dtype=torch.int64, device=self.device)
        ema = torch.empty(self._world * R, dtype=torch.float64, device=self.device)
        age[self._rank * R:(self._rank + 1) * R].copy_(self.age_dev[:R])
        ema[self._rank * R:(self._rank + 1) * R].copy_(self.ema_dev[:R])
        coll.all_gather_rows(age, R)
        coll.all_gather_rows(ema, R)
        return age[:a], ema[:a]

    def adam_struct(self) -> _lib.SSAdamState:
        self.sync_device()
        st = _lib.SSAdamState()
        st.m = self.m_dev.data_ptr()
        st.v = self.v_dev.data_ptr()
        st.grad_ema = self.ema_dev.data_ptr()
        st.age = self.age_dev.data_ptr()
        st.step_count = self.step_count
        return st

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

    def _full(self):
        """(m groups, v groups, age, ema) over all active rows (device)."""
        import torch
        self.sync_device()
        a = self._active
        if self._world == 1:
            return self._groups(self.m_dev), self._groups(self.v_dev), self.age_dev[:a], self.ema_dev[:a]
        coll = parallel.Collectives(self.process_group)
        R, W = self.plan.R, self._world
        out = []
        for flat in (self.m_dev, self.v_dev):
            mine = split_flat(flat, R, self.sh_degree)
            full = {}
            for k, t in mine.items():
                g = torch.empty((W * R,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
                g[self._rank * R:(self._rank + 1) * R].copy_(t)
                coll.all_gather_rows(g, R)
                full[k] = g[:a]
            out.append(full)
        age, ema = self.device_stats()
        return out[0], out[1], age, ema

    def _load_full(self, m, v, age, ema):
        """Keep this rank's rows of full (active-row) state arrays."""
        a = int(age.shape[0])
        self._alloc(a)
        r0, rows = (0, a) if self._world == 1 else (self.plan.row0, self.plan.rows)
        for src, flat in ((m, self.m_dev), (v, self.v_dev)):
            for k, t in self._groups(flat).items():
                t.copy_(src[k][r0:r0 + rows])
        self.age_dev[:rows].copy_(age[r0:r0 + rows])
        self.ema_dev[:rows].copy_(ema[r0:r0 + rows])

    def resize(self, record):
        """Follow a model mutation record (ref optim.py:312-343).  In the
        sharded step every rank applies the same record: the state is gathered,
        remapped and re-split over the new active count."""
        import torch
        kind = type(record).__name__
        a = self._active
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
            return t.clone()

        m, v, age, ema = self._full()
        self._load_full({k: remap(t) for k, t in m.items()}, {k: remap(t) for k, t in v.items()}, remap(age),
                        remap(ema))


class StepWorkspace:
    """Reusable per-model device buffers for step(): the gradient (this
    rank's layout), the per-view losses, and the per-view-slot screen-space
    records of the deferred chain rule (plus their exchange buffers when the
    step is sharded)."""

    def __init__(self, model: DeviceModel):
        import torch
        self.device = model.device
        self.grad = torch.zeros(1, dtype=torch.float32, device=self.device)
        self.loss = torch.zeros(1, dtype=torch.float64, device=self.device)
        self.losses = torch.zeros(1, dtype=torch.float64, device=self.device)
        self._slots = None
        self._recv = None
        # sync-free binning: [0] sticky overflow count, [1] largest pair count
        # (ss_render_opts.bins_status); each step leaves a pinned snapshot
        # checked two steps later (or at once when the loss is read)
        self.bins_status = torch.zeros(2, dtype=torch.int64, device=self.device)
        self.pending = []
        self._snaps = [torch.zeros(2, dtype=torch.int64).pin_memory() for _ in range(8)]
        self._snap_i = 0

    def flush(self):
        """Check every pending step (re-running any that overflowed the
        binning capacity); after this the model holds every step's update."""
        _settle(self, keep=0)

    def prepare(self, grad_elems: int, n_views: int, clear_grad: bool = True):
        import torch
        if self.grad.numel() < max(grad_elems, 1):
            self.grad = torch.zeros(max(grad_elems, 1), dtype=torch.float32, device=self.device)
        if self.losses.numel() < n_views:
            self.losses = torch.zeros(n_views, dtype=torch.float64, device=self.device)
        if clear_grad:  # (else the step's first chain-rule call writes every entry)
            self.grad[:grad_elems].zero_()
        self.losses[:n_views].zero_()
        self.loss.zero_()
        return self.grad[:max(grad_elems, 1)]

    def _buffers(self, attr, slots: int, rows: int):
        import torch
        d = getattr(self, attr)
        if d is None or d[0].shape[0] < slots or d[0].shape[1] < rows:
            cs = max(slots, d[0].shape[0] if d is not None else 0)
            cr = max(rows, 1, d[0].shape[1] if d is not None else 0)
            d = (torch.empty((cs, cr, 9), dtype=torch.float32, device=self.device),
                 torch.empty((cs, cr), dtype=torch.int32, device=self.device))
            setattr(self, attr, d)
        return [(d[0][i, :rows], d[1][i, :rows]) for i in range(slots)]

    def slot_records(self, slots: int, rows: int):
        """Per view slot: g9 (rows, 9) float32 and rinv (rows,) int32."""
        return self._buffers("_slots", slots, rows)

    def recv_records(self, slots: int, rows: int):
        return self._buffers("_recv", slots, rows)

    def defer_buffers(self, views: int, n_in: int, device=None):
        """(g9 list, rinv list) of `views` slots over n_in rows (ss_backward's defer=)."""
        recs = self.slot_records(views, n_in)
        return [g for g, _ in recs], [r for _, r in recs]


CHAIN_MAX_VIEWS = 16  # ss_chain_views
# concurrent view lanes of a step (streams; see _DeviceKernels._lane)
VIEW_LANES = max(1, int(os.environ.get("SS_VIEW_LANES", "4")))


def chain_views(model: DeviceModel, views, g9, rinv, grad, subset_tensor=None, j0=0, j1=None, row0=0, rows=None,
                ld=None, init=False):
    """The deferred chain rule of `views` (their backward_device calls got
    defer=(g9[i], rinv[i])): one pass over the rows, the gradient read and
    written once (ss_chain_views_range).  g9 / rinv entries are tensors or
    raw device addresses."""
    import ctypes as C
    c = _lib.ctx(model.device.index)
    k = len(views)
    cams = (_lib.SSCamera * k)(*[camera_struct(v.pose, v.intrinsics) for v in views])
    lights = (_lib.SSLight * k)(*[light_struct(v.light_state) for v in views])
    addr = lambda x: x if isinstance(x, int) else x.data_ptr()
    gp = (C.c_void_p * k)(*[addr(g9[i]) for i in range(k)])
    rp = (C.c_void_p * k)(*[addr(rinv[i]) for i in range(k)])
    if j1 is None:
        j1 = int(subset_tensor.numel()) if subset_tensor is not None else model.count
    a = model.active_count
    rows = a if rows is None else rows
    ld = a if ld is None else ld
    # init: the gradient rows were not cleared; every entry gets written (ss_chain_views_range_init)
    c.check(c.lib.ss_chain_views_range_init(c.handle, model.struct(), cams, lights, k, gp, rp,
                                            _lib.ptr(subset_tensor) if subset_tensor is not None else None,
                                            int(j0), int(j1), int(row0), int(rows), _lib.ptr(grad), int(ld),
                                            1 if init else 0))


def _row_struct(dm: DeviceModel, row0: int, rows: int) -> _lib.SSModel:
    """ss_model of rows [row0, row0 + rows) of dm, all of them active (a row
    shard for the sharded Adam)."""
    s = dm.struct()
    B = (dm.sh_degree + 1) ** 2
    for k, w, es in (("means", 3, 4), ("log_scales", 3, 4), ("quaternions", 4, 4), ("logit_opacities", 1, 4),
                     ("sh_coeffs", 3 * B, 4), ("light_visibility", 1, 4), ("object_ids", 1, 4)):
        setattr(s, k, getattr(dm, k).data_ptr() + row0 * w * es)
    s.count = rows
    s.active_count = rows
    return s


class _DeviceKernels:
    """The compute of parallel.sharded_step on this GPU (libsplat_b200)."""

    def __init__(self, dm: DeviceModel, state: OptimizerState, ws: StepWorkspace, views, subset, extent_cutoff,
                 plan: parallel.ShardPlan, deterministic=True, p2p=False):
        self.dm, self.state, self.ws, self.sub, self.cutoff, self.plan = dm, state, ws, subset, extent_cutoff, plan
        self.deterministic = deterministic
        self.p2p = p2p and plan.world > 1
        self.window = None
        self.n_in = int(subset.numel()) if subset is not None else dm.count
        B = (dm.sh_degree + 1) ** 2
        self.ld = dm.active_count if plan.world == 1 else plan.R
        # without a row subset the first chain-rule call initialises the
        # gradient (no clear of the 59-float rows, no first read of them)
        self.init_chain = subset is None
        self.grad = ws.prepare(self.ld * (11 + 3 * B), len(views), clear_grad=not self.init_chain)
        self.gts = {}
        self.views = views
        self.lanes = None
        self._n_local = 0
        self._view_lane = {}

    def stage(self, local_views):
        gts = _stage_ground_truth(local_views, self.dm.device)
        self.gts = {id(v): g for v, g in zip(local_views, gts)}

    def _rows_alloc(self):
        return self.n_in if self.plan.world == 1 else max(self.plan.padded, self.dm.count)

    def records(self, slots):
        return self.ws.slot_records(slots, self._rows_alloc())

    def _lane(self, t):
        """(stream, context) of the t-th local view: views alternate over
        VIEW_LANES streams, each with its own library context (scratch
        arena), so one view's latency-bound preprocess / sorts / binning
        overlap the previous view's blend kernels.  Lane 0 is the caller's
        stream; the others fork from it at the first view (join())."""
        import torch
        L = VIEW_LANES
        dev = self.dm.device
        if self.lanes is None:
            cur = torch.cuda.current_stream(dev)
            self.lanes = [(cur, None)]
            for k in range(1, L):
                ls = _lib.lane_stream(dev.index, k)
                ls.wait_stream(cur)
                self.lanes.append((ls, None))
        return t % L, self.lanes[t % L][0]

    def join(self):
        """The caller's stream waits for every view lane."""
        import torch
        if self.lanes is None:
            return
        cur = self.lanes[0][0]
        for s, _ in self.lanes[1:]:
            cur.wait_stream(s)
        self.lanes = None

    def backward(self, view, rec, i):
        import torch
        k, stream = self._lane(self._n_local)
        self._n_local += 1
        # a view object passed twice keeps its first lane: its per-camera tile
        # hint / order buffers are then written in stream order
        k0 = self._view_lane.setdefault(id(view), k)
        if k0 != k:
            k, stream = k0, self.lanes[k0][0]
        with torch.cuda.stream(stream):
            self._backward(view, rec, i, _lib.lane_ctx(self.dm.device.index, k))

    def _backward(self, view, rec, i, ctx):
        import torch
        g9, rinv = rec
        sharded_subset = self.plan.world > 1 and self.sub is not None
        if sharded_subset:  # input-indexed records first, then scattered to row order for the exchange
            tmp_g9 = torch.empty((self.n_in, 9), dtype=torch.float32, device=self.dm.device)
            tmp_r = torch.empty(self.n_in, dtype=torch.int32, device=self.dm.device)
            defer = (tmp_g9, tmp_r)
        else:
            defer = (g9[:self.n_in], rinv[:self.n_in])
        backward_device(self.dm, view, self.grad, self.ws.losses[i:i + 1], None, self.cutoff, 0, None,
                        subset_tensor=self.sub, gt=self.gts[id(view)], defer=defer, deterministic=self.deterministic,
                        bins_status=self.ws.bins_status, ctx=ctx)
        if sharded_subset:
            rinv.fill_(-1)
            g9[self.sub] = tmp_g9
            rinv[self.sub] = tmp_r

    def invisible(self, rec):
        rec[1].fill_(-1)  # 0xffffffff: not visible in this view

    def _peer_window(self, coll):
        """Every rank's slot record buffers and parameter columns, mapped
        into this process (parallel.PeerWindow; re-shared when reallocated)."""
        d = self.ws._slots
        tensors = {"g9": d[0], "rinv": d[1]}
        tensors.update({k: getattr(self.dm, k) for k in TRAINABLE})
        win = getattr(self.ws, "_window", None)
        if win is None or win.key != parallel.PeerWindow.key_of(tensors):
            win = self.ws._window = parallel.PeerWindow(coll.group, tensors)
        return win

    def exchange(self, coll, send):
        if self.p2p:
            # zero-copy: the chain rule reads each rank's records from that
            # rank's HBM; first every rank's records must be complete
            self.window = self._peer_window(coll)
            coll.barrier()
            return list(range(len(send)))
        P = self.plan.padded
        recv = self.ws.recv_records(len(send), P)
        for (sg, sr), (rg, rr) in zip(send, recv):
            coll.all_to_all(rg, sg[:P])
            coll.all_to_all(rr, sr[:P])
        return recv

    def shard_view(self, rec, s):
        """Source rank s's records of this rank's rows, as addresses indexed by row."""
        if self.p2p:  # rec = the view slot: rank s's own (row-indexed) buffer, mapped here
            peer = self.window.peers[s]
            return (peer["g9"][rec].data_ptr(), peer["rinv"][rec].data_ptr())
        R, r0 = self.plan.R, self.plan.row0
        g9, rinv = rec
        return (g9.data_ptr() + (s * R - r0) * 36, rinv.data_ptr() + (s * R - r0) * 4)

    def chain_batch(self, views, recs):
        if self.dm.active_count == 0 or self.n_in == 0 or self.plan.rows == 0:
            return
        g9 = [r[0] for r in recs]
        rinv = [r[1] for r in recs]
        init, self.init_chain = self.init_chain, False  # the first batch initialises the gradient
        if self.plan.world == 1:
            chain_views(self.dm, views, g9, rinv, self.grad, self.sub, init=init)
        else:
            r0, rows = self.plan.row0, self.plan.rows
            chain_views(self.dm, views, g9, rinv, self.grad, None, j0=r0, j1=r0 + rows, row0=r0, rows=rows,
                        ld=self.ld, init=init)

    def sum_losses(self, coll):
        V = len(self.views)
        losses = self.ws.losses[:V]
        if coll is not None:  # each entry is non-zero on exactly one rank: the sum is exact
            coll.all_reduce_(losses)
            coll.all_reduce_(self.ws.bins_status[:1], "max")  # any rank's binning overflow voids the step everywhere
        c = _lib.ctx(self.dm.device.index)
        c.check(c.lib.ss_sum_f64(c.handle, losses.data_ptr(), V, self.ws.loss.data_ptr()))
        return self.ws.loss

    def adam(self, n_views):
        st = self.state
        if self.dm.active_count == 0:  # frozen-only model: no state change (optim.py:374)
            return
        c = _lib.ctx(self.dm.device.index)
        ast = st.adam_struct()
        ast.skip_if = self.ws.bins_status.data_ptr()  # a step whose binning overflowed leaves the model alone
        if self.plan.world == 1:
            ms = self.dm.struct()
        else:
            ms = _row_struct(self.dm, self.plan.row0, self.plan.rows)
        if self.p2p and self.plan.rows > 0:
            # the parameter all-gather fused into the update: every row is
            # also stored into each other rank's replica (peer memory)
            import ctypes as C
            B = (self.dm.sh_degree + 1) ** 2
            widths = dict(means=3, log_scales=3, quaternions=4, logit_opacities=1, sh_coeffs=3 * B)
            rows = []
            for r, peer in enumerate(self.window.peers):
                if r == self.plan.rank:
                    continue
                rows += [peer[k].data_ptr() + self.plan.row0 * widths[k] * 4 for k in TRAINABLE]
            ptrs = (C.c_void_p * len(rows))(*rows)
            c.check(c.lib.ss_adam_step_peers(c.handle, ms, ast, self.grad.data_ptr(), self.ld, n_views, st.hparams(),
                                             self.plan.world - 1, ptrs))
        else:
            c.check(c.lib.ss_adam_step_ld(c.handle, ms, ast, self.grad.data_ptr(), self.ld, n_views, st.hparams()))
        st.step_count = int(ast.step_count)
        st._host = None  # device moments changed: the host mirror is stale

    def gather(self, coll):
        if self.p2p:  # Adam already stored every row into every replica: order it before any next use
            coll.barrier()
            return
        R = self.plan.R
        for k in TRAINABLE:
            t = getattr(self.dm, k)
            view, write_back = parallel.padded_rows_view(t, self.plan.padded)
            coll.all_gather_rows(view, R)
            if write_back is not None:
                write_back()


def step(model, state: OptimizerState, views, index_subset=None, extent_cutoff: bool = True, precision: int = 0,
         process_group=None, workspace: Optional[StepWorkspace] = None, sync_loss: bool = True,
         deterministic: bool = True, exchange: Optional[str] = None):
    """ref optim.py:353 -- one Adam step over the ready views; returns the mean loss.

    With a `process_group` (or a state created with one) every rank passes
    the SAME views; rank r renders views r, r+N, ... and the step is sharded
    as parallel.py describes -- bit-identical to the single-GPU step.
    `sync_loss=False` returns the device loss tensor instead of a host float
    (no host synchronisation).  `deterministic=False` selects the backward's
    throughput mode: per-(tile, splat) sums added with float atomics instead
    of the fixed-order partial sums (reruns may differ in the last bits).
    `exchange` (sharded steps): "p2p" -- the chain rule reads the other
    ranks' records from their memory and Adam stores the updated rows into
    every replica (CUDA IPC peer memory; the default on NCCL groups) -- or
    "collectives" (an all-to-all and an all-gather; the default otherwise).

    The fp32 path bins without reading pair counts back (sync-free; see
    ss_render_opts.bins_status): each step leaves a snapshot of its binning
    status, checked when its loss is read or two steps later.  A step whose
    pairs outgrew the capacity left the model untouched (its Adam is skipped
    on the device, and every later step until the check); the check raises
    the capacity and re-runs those steps in order, so the trajectory is the
    same as without the capacity limit.
    """
    ready = [v for v in views if v.ready]
    if not ready:
        raise ValueError("no ready views")
    if state.active_count != model.active_count:
        raise ValueError("optimizer state out of sync with model")
    pg = process_group if process_group is not None else state.process_group
    if pg is not None and pg is not state.process_group:
        raise ValueError("the optimizer state was created for a different process group")
    dm, uploaded = as_device(model, keep_f64=precision == 1)
    a = dm.active_count
    sub = _subset_tensor(index_subset, dm.device)
    persistent = workspace is not None
    ws = workspace if persistent else StepWorkspace(dm)
    if precision != 0:
        if state.plan.world > 1:
            raise ValueError("the fp64 blend (precision=1) is single-GPU")
        loss = _step_immediate(dm, state, ready, sub, extent_cutoff, precision, ws, deterministic)
    else:
        _settle(ws, keep=1)  # the step before last: checked (and re-run after an overflow)
        if exchange is None:
            exchange = ("p2p" if (pg is not None and _backend(pg) == "nccl" and parallel.peer_access_ok(pg))
                        else "collectives")
        if exchange not in ("p2p", "collectives"):
            raise ValueError(f"unknown exchange {exchange!r}")
        args = (dm, state, ready, sub, extent_cutoff, pg, deterministic, exchange == "p2p")
        loss = _step_binned(ws, *args)
        _note(ws, args)
        if sync_loss or not persistent:
            loss.item()  # the device is idle after this: the check costs no extra wait
            _settle(ws, keep=0)
            loss = ws.loss
    if uploaded and a > 0:
        dm.write_back(model, TRAINABLE, rows=a)
    total = len(ready)
    if not sync_loss:
        return loss / total
    return float(loss.item()) / total


def _backend(pg):
    import torch.distributed as dist
    return dist.get_backend(pg)


def _step_binned(ws, dm, state, ready, sub, extent_cutoff, pg, deterministic, p2p=False):
    plan = state.plan
    kern = _DeviceKernels(dm, state, ws, ready, sub, extent_cutoff, plan, deterministic, p2p)
    kern.stage(parallel.shard_views(ready, plan.rank, plan.world) if plan.world > 1 else ready)
    coll = parallel.Collectives(pg) if plan.world > 1 else None
    return parallel.sharded_step(kern, ready, plan, coll, CHAIN_MAX_VIEWS)


def _note(ws, args):
    """Snapshot this step's binning status into pinned memory (no wait)."""
    import torch
    snap = ws._snaps[ws._snap_i % len(ws._snaps)]  # a ring: at most 2 steps are pending
    ws._snap_i += 1
    snap.copy_(ws.bins_status, non_blocking=True)
    ev = torch.cuda.Event()
    ev.record()
    step_count_after = args[1].step_count
    ws.pending.append((ev, snap, args, step_count_after))


def _settle(ws, keep):
    """Check the pending steps but the newest `keep`; after an overflow,
    raise the pair capacity and re-run the voided steps in order."""
    while len(ws.pending) > keep:
        ev, snap, args, count_after = ws.pending[0]
        ev.synchronize()
        if int(snap[0]) == 0:
            ws.pending.pop(0)
            continue
        _recover(ws)
        return


def _recover(ws):
    """The oldest pending step overflowed its pair buffers (and every later
    pending step was skipped on the device): grow, clear, re-run them all."""
    import torch
    torch.cuda.synchronize()
    redo = ws.pending
    ws.pending = []
    st = ws.bins_status.cpu()
    dev = redo[0][2][0].device
    need = int(st[1])
    _lib.pair_capacity(dev.index, need + need // 4 + 65536)
    ws.bins_status.zero_()
    state = redo[0][2][1]
    # every pending step left the state alone: restart from the first one's count
    state.step_count = redo[0][3] - 1
    for _, _, args, _ in redo:
        _step_binned(ws, *args)
        _note(ws, args)
    torch.cuda.synchronize()
    _settle(ws, keep=0)


def _step_immediate(dm, state, ready, sub, extent_cutoff, precision, ws, deterministic=True):
    """Per-view chain rule into the gradient (the fp64 blend instantiation)."""
    B = (dm.sh_degree + 1) ** 2
    a = dm.active_count
    grad = ws.prepare(a * (11 + 3 * B), len(ready))
    gts = _stage_ground_truth(ready, dm.device)
    for i, (v, gt) in enumerate(zip(ready, gts)):
        backward_device(dm, v, grad, ws.losses[i:i + 1], None, extent_cutoff, precision, None, subset_tensor=sub, gt=gt,
                        deterministic=deterministic)
    c = _lib.ctx(dm.device.index)
    c.check(c.lib.ss_sum_f64(c.handle, ws.losses.data_ptr(), len(ready), ws.loss.data_ptr()))
    if a > 0:
        ast = state.adam_struct()
        c.check(c.lib.ss_adam_step(c.handle, dm.struct(), ast, grad.data_ptr(), len(ready), state.hparams()))
        state.step_count = int(ast.step_count)
        state._host = None
    return ws.loss
