"""Pool maintenance on the GPU: drop-in for the row
bookkeeping the server runs every tick -- ref pkg/src/splatstream/model.py
(GridIndex.rebuild, freeze_range, prune_rows, apply_mutation, the mutation
records), expansion.py (freeze_policy, precull, prune) and
protocol/packets.py (encode_ordering) -- on a DeviceModel.

Row selection, row moves, the grid and the permutation varints run in
csrc/ss_pool.cu; results equal the reference's (tests/test_pool.py, against
outcomes of the unmodified reference).  Records carry host numpy arrays, as
in the reference, because they travel in ordering packets.
"""

from __future__ import annotations

import struct
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import _lib
from .model import DeviceModel
from .render import camera_struct


# ---------------------------------------------------------------- records (ref model.py:36-62)
@dataclass
class PermuteRecord:
    """Row reorder: new_row[i] = old_row[permutation[i]]."""
    permutation: np.ndarray
    new_active_count: int


@dataclass
class AppendRecord:
    """`count` rows inserted at `insert_at` (in front of the frozen region)."""
    insert_at: int
    count: int
    object_ids: np.ndarray
    new_active_count: int


@dataclass
class PruneRecord:
    """Rows at `indices` (pre-compaction numbering) removed."""
    indices: np.ndarray
    new_active_count: int


def _ctx(model):
    c = _lib.ctx(model.device.index)
    c.bind_stream()
    return c


def _select(model: DeviceModel, s: _lib.SSSelect, as_tensor: bool = False):
    import torch
    out = torch.empty(max(int(s.n), 1), dtype=torch.int64, device=model.device)
    cnt = _lib.i64(0)
    c = _ctx(model)
    c.check(c.lib.ss_select_rows(c.handle, s, out.data_ptr(), C_byref(cnt)))
    if as_tensor:  # the rows stay on the device (ascending)
        return out[:cnt.value]
    return out[:cnt.value].cpu().numpy()


def C_byref(x):
    import ctypes
    return ctypes.byref(x)


def freeze_policy(model: DeviceModel, optimizer_stats, age_threshold: int = 100,
                  grad_threshold: float = 1e-4) -> np.ndarray:
    """ref expansion.py:134-142 -- active rows with age >= threshold and grad-EMA < threshold."""
    s = _lib.SSSelect()
    s.kind = 0
    if hasattr(optimizer_stats, "device_stats"):  # an OptimizerState (device buffers, gathered if sharded)
        age, ema = optimizer_stats.device_stats()
    else:  # any object with device age / grad_ema tensors
        age, ema = optimizer_stats.age, optimizer_stats.grad_ema
    s.n = int(age.shape[0])
    s.age = age.data_ptr()
    s.grad_ema = ema.data_ptr()
    s.age_threshold = int(age_threshold)
    s.grad_threshold = float(grad_threshold)
    return _select(model, s)


def _gather(model: DeviceModel, row_map: np.ndarray, new_active: int, fill: Optional[DeviceModel] = None):
    """Replace every column by its rows `row_map` (negative: placeholder rows)."""
    import torch
    n = int(row_map.size)
    dev = model.device
    B = (model.sh_degree + 1) ** 2
    dst = DeviceModel(torch.empty((n, 3), dtype=torch.float32, device=dev),
                      torch.empty((n, 3), dtype=torch.float32, device=dev),
                      torch.empty((n, 4), dtype=torch.float32, device=dev),
                      torch.empty(n, dtype=torch.float32, device=dev),
                      torch.empty((n, 3, B), dtype=torch.float32, device=dev),
                      torch.empty(n, dtype=torch.float32, device=dev),
                      torch.empty(n, dtype=torch.int32, device=dev), new_active, model.sh_degree)
    if n:
        m = torch.from_numpy(np.ascontiguousarray(row_map, dtype=np.int64)).to(dev)
        c = _ctx(model)
        fs = fill.struct() if fill is not None else None
        c.check(c.lib.ss_gather_rows(c.handle, model.struct(), dst.struct(), m.data_ptr(), n, fs))
    for k in ("means", "log_scales", "quaternions", "logit_opacities", "sh_coeffs", "light_visibility", "object_ids"):
        setattr(model, k, getattr(dst, k))
    model.active_count = int(new_active)


def permute(model: DeviceModel, permutation, new_active_count: int):
    """GaussianModel.permute (ref model.py:153-158) on the device."""
    permutation = np.asarray(permutation)
    if not np.array_equal(np.sort(permutation.astype(np.int64)), np.arange(model.count)):
        raise ValueError("not a permutation of current rows")
    _gather(model, permutation.astype(np.int64), new_active_count)


def remove_rows(model: DeviceModel, indices, new_active_count: int):
    """GaussianModel.remove_rows (ref model.py:160-164)."""
    keep = np.ones(model.count, dtype=bool)
    keep[np.asarray(indices, dtype=np.int64)] = False
    _gather(model, np.flatnonzero(keep).astype(np.int64), new_active_count)


def freeze_range(model: DeviceModel, indices) -> Optional[PermuteRecord]:
    """ref model.py:207-228: kept actives, newly frozen, previously frozen."""
    idx = np.unique(np.asarray(list(indices), dtype=np.int64))
    if idx.size == 0:
        return None
    if (idx >= model.active_count).any() or (idx < 0).any():
        raise ValueError("freeze targets must be active rows")
    mask = np.zeros(model.count, dtype=bool)
    mask[idx] = True
    kept = np.nonzero(~mask[: model.active_count])[0]
    frozen_tail = np.arange(model.active_count, model.count)
    permutation = np.concatenate([kept, idx, frozen_tail])
    new_active = kept.size
    _gather(model, permutation, new_active)
    return PermuteRecord(permutation=permutation, new_active_count=new_active)


def prune_rows(model: DeviceModel, indices) -> Optional[PruneRecord]:
    """ref model.py:231-240."""
    idx = np.unique(np.asarray(indices, dtype=np.int64))
    if idx.size == 0:
        return None
    if (idx < 0).any() or (idx >= model.count).any():
        raise ValueError("prune index out of range")
    removed_active = int((idx < model.active_count).sum())
    new_active = model.active_count - removed_active
    remove_rows(model, idx, new_active)
    return PruneRecord(indices=idx, new_active_count=new_active)


def prune(model: DeviceModel, opacity_floor: float = 0.01):
    """ref expansion.py:184-197 -- (removed pre-compaction indices, PruneRecord or None)."""
    if not 0 <= opacity_floor < 1:
        raise ValueError("opacity_floor must be in [0, 1)")
    s = _lib.SSSelect()
    s.kind = 1
    s.n = int(model.active_count)
    s.logits = model.logit_opacities.data_ptr()
    s.opacity_floor = float(opacity_floor)
    removed = _select(model, s) if s.n else np.zeros(0, np.int64)
    record = prune_rows(model, removed) if removed.size else None
    return removed, record


def _placeholders(n: int, sh_degree: int, device):
    """ref model.py:243-256 placeholder_batch (one row; object ids set afterwards)."""
    import torch
    B = (sh_degree + 1) ** 2
    return DeviceModel(torch.zeros((1, 3), dtype=torch.float32, device=device),
                       torch.full((1, 3), -10.0, dtype=torch.float32, device=device),
                       torch.tensor([[1.0, 0.0, 0.0, 0.0]], dtype=torch.float32, device=device),
                       torch.full((1,), -100.0, dtype=torch.float32, device=device),
                       torch.zeros((1, 3, B), dtype=torch.float32, device=device),
                       torch.ones(1, dtype=torch.float32, device=device),
                       torch.zeros(1, dtype=torch.int32, device=device), 1, sh_degree)


def apply_mutation(model: DeviceModel, record) -> None:
    """ref model.py:259-292: replay a server-side row mutation on a device replica."""
    import torch
    if isinstance(record, PermuteRecord) or type(record).__name__ == "PermuteRecord":
        if not 0 <= record.new_active_count <= model.count:
            raise ValueError("permute record active count out of range")
        permute(model, record.permutation, record.new_active_count)
    elif isinstance(record, AppendRecord) or type(record).__name__ == "AppendRecord":
        if record.insert_at != model.active_count:
            raise ValueError("append record does not start at the active boundary")
        if record.new_active_count != record.insert_at + len(record.object_ids):
            raise ValueError("append record counts disagree")
        at, cnt, n = int(record.insert_at), len(record.object_ids), model.count
        row_map = np.concatenate([np.arange(at), -1 - np.zeros(cnt, np.int64), np.arange(at, n)]).astype(np.int64)
        _gather(model, row_map, record.new_active_count, _placeholders(cnt, model.sh_degree, model.device))
        if cnt:
            model.object_ids[at:at + cnt] = torch.from_numpy(np.asarray(record.object_ids, np.int32)).to(model.device)
    elif isinstance(record, PruneRecord) or type(record).__name__ == "PruneRecord":
        idx = np.unique(np.asarray(record.indices, dtype=np.int64))
        if idx.size and (int(idx.max()) >= model.count or int(idx.min()) < 0):
            raise ValueError("prune record outside replica rows")
        removed_active = int((idx < model.active_count).sum())
        if record.new_active_count != model.active_count - removed_active:
            raise ValueError("prune record counts disagree")
        remove_rows(model, idx, record.new_active_count)
    else:
        raise TypeError(f"unknown record {type(record)}")


def baselines_apply_record(baselines, record) -> None:
    """DeltaBaselines.apply_record (ref protocol/delta.py:237-256) on device baselines."""
    import torch
    for name in ("means", "log_scales"):
        arr = getattr(baselines, name)
        kind = type(record).__name__
        if kind == "PermuteRecord":
            arr = arr[torch.from_numpy(np.asarray(record.permutation, np.int64)).to(arr.device)].clone()
        elif kind == "AppendRecord":
            pad = torch.zeros((int(record.count),) + tuple(arr.shape[1:]), dtype=arr.dtype, device=arr.device)
            arr = torch.cat([arr[:record.insert_at], pad, arr[record.insert_at:]])
        elif kind == "PruneRecord":
            keep = np.ones(arr.shape[0], dtype=bool)
            keep[np.asarray(record.indices, np.int64)] = False
            arr = arr[torch.from_numpy(np.flatnonzero(keep)).to(arr.device)].clone()
        else:
            raise TypeError(f"unknown record {type(record)}")
        setattr(baselines, name, arr)


# ---------------------------------------------------------------- grid + precull
class GridIndex:
    """ref model.py:383-429 with the rebuild on the device.  `cell_map` (dict
    cell -> member rows, first-appearance order) is materialised on demand."""

    def __init__(self, cell_size: float = 2.0, origin=(0.0, 0.0, 0.0)):
        if cell_size <= 0:
            raise ValueError("cell_size must be positive")
        self.cell_size = float(cell_size)
        self.origin = np.asarray(origin, dtype=np.float64)
        self.initialized_cells: set = set()
        self.cells = None       # (n, 3) int64 device: cell of every row at the last rebuild
        self.cell_keys = None   # (C, 3) int64 device, dict order
        self.cell_lens = None   # (C,) int64 device
        self.cell_rows = None   # (n,) int64 device, members grouped by cell
        self._map = {}

    def cell_of(self, position):
        c = np.floor((np.asarray(position, dtype=np.float64) - self.origin) / self.cell_size)
        return (int(c[0]), int(c[1]), int(c[2]))

    def cells_of(self, positions):
        return np.floor((np.asarray(positions, dtype=np.float64) - self.origin) / self.cell_size).astype(np.int64)

    def cell_center(self, cell):
        return self.origin + (np.asarray(cell, dtype=np.float64) + 0.5) * self.cell_size

    @property
    def cell_diagonal(self) -> float:
        return float(self.cell_size * np.sqrt(3.0))

    def rebuild(self, model: DeviceModel):
        import torch
        self._map = None
        n = model.count
        dev = model.device
        self.cells = torch.empty((max(n, 1), 3), dtype=torch.int64, device=dev)[:n]
        self.cell_keys = torch.empty((max(n, 1), 3), dtype=torch.int64, device=dev)
        self.cell_lens = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
        self.cell_rows = torch.empty(max(n, 1), dtype=torch.int64, device=dev)[:n]
        g = _lib.SSGridSpec()
        g.origin = _lib.f64arr(self.origin, 3)
        g.cell_size = self.cell_size
        nc = _lib.i64(0)
        c = _ctx(model)
        c.check(c.lib.ss_grid_rebuild(c.handle, model.means.data_ptr() if n else None, n, g,
                                      self.cells.data_ptr() if n else None, self.cell_keys.data_ptr(),
                                      self.cell_lens.data_ptr(), self.cell_rows.data_ptr() if n else None,
                                      C_byref(nc)))
        self.cell_keys = self.cell_keys[:nc.value]
        self.cell_lens = self.cell_lens[:nc.value]

    @property
    def cell_map(self) -> dict:
        if self._map is None:
            keys = self.cell_keys.cpu().numpy() if self.cell_keys is not None else np.zeros((0, 3), np.int64)
            lens = self.cell_lens.cpu().numpy() if self.cell_lens is not None else np.zeros(0, np.int64)
            rows = self.cell_rows.cpu().numpy() if self.cell_rows is not None else np.zeros(0, np.int64)
            off = np.concatenate([[0], np.cumsum(lens)])
            self._map = {tuple(int(v) for v in keys[i]): rows[off[i]:off[i + 1]].tolist() for i in range(len(lens))}
        return self._map

    def mark_initialized(self, cell):
        self.initialized_cells.add(tuple(int(v) for v in cell))


def precull(model: DeviceModel, grid: GridIndex, poses: Sequence, intr, depth_buffers=None, as_tensor: bool = False):
    """ref expansion.py:145-181 on the device: rows (as of the grid's last
    rebuild) whose cell passes the conservative frustum test in any camera,
    with the engine-depth occlusion test when depth buffers are given.
    as_tensor=True keeps the rows on the device (a CUDA int64 tensor, the
    optimizer step's index_subset without a round trip through the host)."""
    import torch
    if grid.cells is None or grid.cells.shape[0] == 0:
        if as_tensor:
            return torch.zeros(0, dtype=torch.int64, device=model.device)
        return np.zeros(0, dtype=np.int64)
    cams = (_lib.SSPoolCamera * max(len(poses), 1))()
    keep_alive = []
    tx = (intr.width / 2.0) / intr.fx
    ty = (intr.height / 2.0) / intr.fy
    nx = 1.0 / np.sqrt(1.0 + tx * tx)
    ny = 1.0 / np.sqrt(1.0 + ty * ty)
    if depth_buffers is None:
        depth_buffers = [None] * len(poses)
    for i, (pose, depth) in enumerate(zip(poses, depth_buffers)):
        cs = camera_struct(pose, intr)
        cc = cams[i]
        cc.position, cc.rot_cw = cs.position, cs.rot_cw
        cc.fx, cc.fy, cc.cx, cc.cy = cs.fx, cs.fy, cs.cx, cs.cy
        cc.near_plane, cc.far_plane = float(intr.near), float(intr.far)
        cc.tx, cc.ty, cc.nx, cc.ny = float(tx), float(ty), float(nx), float(ny)
        cc.width, cc.height = int(intr.width), int(intr.height)
        if depth is not None:
            d = torch.as_tensor(np.ascontiguousarray(depth, np.float64), device=model.device) \
                if not isinstance(depth, torch.Tensor) else depth.to(model.device, torch.float64).contiguous()
            keep_alive.append(d)
            cc.depth = d.data_ptr()
    s = _lib.SSSelect()
    s.kind = 2
    s.n = int(grid.cells.shape[0])
    s.cells = grid.cells.data_ptr()
    s.origin = _lib.f64arr(grid.origin, 3)
    s.cell_size = grid.cell_size
    s.margin = grid.cell_diagonal / 2.0
    s.n_cameras = len(poses)
    s.cameras = cams
    out = _select(model, s, as_tensor)
    if not as_tensor:
        torch.cuda.current_stream(model.device).synchronize()
    return out


# ---------------------------------------------------------------- ordering packet (ref protocol/packets.py:145-180)
_KIND_PERMUTE, _KIND_APPEND, _KIND_PRUNE = 0, 1, 2


def _varints_host(values) -> bytes:
    out = bytearray()
    for n in np.asarray(values, dtype=np.uint64).reshape(-1):
        n = int(n)
        while True:
            b = n & 0x7F
            n >>= 7
            if n:
                out.append(b | 0x80)
            else:
                out.append(b)
                break
    return bytes(out)


def encode_ordering(records, device=None) -> bytes:
    """ref packets.py:160-180; permutation blocks (zigzag offsets from the
    identity as LEB128, the bulk of the packet) are encoded on the device,
    then deflated on the host (zlib level 6, as the reference)."""
    import ctypes
    import torch
    from .protocol import host_zlib
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    out = [struct.pack("<I", len(records))]
    for rec in records:
        kind = type(rec).__name__
        if kind == "PermuteRecord":
            perm = np.asarray(rec.permutation, dtype=np.int64)
            n = perm.size
            raw = b""
            if n:
                p = torch.from_numpy(perm).to(dev)
                buf = torch.empty(10 * n, dtype=torch.uint8, device=dev)
                ln = _lib.u64(0)
                c = _lib.ctx(dev.index)
                c.bind_stream()
                c.check(c.lib.ss_zigzag_varints(c.handle, p.data_ptr(), n, buf.data_ptr(), buf.numel(),
                                                 ctypes.byref(ln)))
                raw = buf[:ln.value].cpu().numpy().tobytes()
            blob = host_zlib(raw)
            out.append(struct.pack("<BIII", _KIND_PERMUTE, n, rec.new_active_count, len(blob)))
            out.append(blob)
        elif kind == "AppendRecord":
            oids = np.asarray(rec.object_ids, dtype=np.int64)
            out.append(struct.pack("<BIII", _KIND_APPEND, rec.insert_at, rec.count, rec.new_active_count))
            out.append(_varints_host(oids))
        elif kind == "PruneRecord":
            idx = np.asarray(rec.indices, dtype="<u4")
            out.append(struct.pack("<BII", _KIND_PRUNE, idx.size, rec.new_active_count))
            out.append(idx.tobytes())
        else:
            raise TypeError(f"unknown record {type(rec)}")
    return b"".join(out)


__all__ = ["AppendRecord", "GridIndex", "PermuteRecord", "PruneRecord", "apply_mutation", "baselines_apply_record",
           "encode_ordering", "freeze_policy", "freeze_range", "permute", "precull", "prune", "prune_rows",
           "remove_rows"]
