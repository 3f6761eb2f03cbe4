"""Rigid dynamic objects on a DeviceModel (ref model.py:326-404 ObjectRegistry).

Rows with object_id k > 0 satisfy world_mean = R_k local_mean + t_k and
world_quat = q_k * local_quat.  The registry keeps the row-aligned local
poses in HBM (float64, like the reference's arrays) and rewrites or
re-derives them with the library's kernels (`ss_apply_object_transform`,
`ss_refresh_object_locals[_rows]`); transforms stay on the host, as small
dicts.  Same method names and arguments as the reference.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .geometry import quat_normalize
from .model import DeviceModel
from .pool import AppendRecord, PermuteRecord, PruneRecord


class ObjectRegistry:
    def __init__(self, device=None):
        import torch
        self.transforms: dict = {}  # object_id -> (quaternion wxyz, translation), float64
        self._dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.local_means = torch.zeros((0, 3), dtype=torch.float64, device=self._dev)
        self.local_rotations = torch.zeros((0, 4), dtype=torch.float64, device=self._dev)

    def set_transform(self, object_id: int, quat, translation):
        self.transforms[int(object_id)] = (quat_normalize(np.asarray(quat, dtype=np.float64)),
                                           np.asarray(translation, dtype=np.float64))

    def get_transform(self, object_id: int):
        return self.transforms.get(int(object_id), (np.array([1.0, 0, 0, 0]), np.zeros(3)))

    def resize(self, record):
        """Follow a mutation record (ref model.py:350-369)."""
        import torch
        if isinstance(record, PermuteRecord):
            perm = torch.as_tensor(np.asarray(record.permutation, np.int64), device=self._dev)
            self.local_means = self.local_means[perm].contiguous()
            self.local_rotations = self.local_rotations[perm].contiguous()
        elif isinstance(record, AppendRecord):
            at, k = int(record.insert_at), int(record.count)
            ident = torch.tensor([1.0, 0, 0, 0], dtype=torch.float64, device=self._dev).repeat(k, 1)
            self.local_means = torch.cat([self.local_means[:at], torch.zeros((k, 3), dtype=torch.float64,
                                                                             device=self._dev),
                                          self.local_means[at:]])
            self.local_rotations = torch.cat([self.local_rotations[:at], ident, self.local_rotations[at:]])
        elif isinstance(record, PruneRecord):
            keep = torch.ones(self.local_means.shape[0], dtype=torch.bool, device=self._dev)
            keep[torch.as_tensor(np.asarray(record.indices, np.int64), device=self._dev)] = False
            self.local_means = self.local_means[keep].contiguous()
            self.local_rotations = self.local_rotations[keep].contiguous()
        else:
            raise TypeError(f"unknown record {type(record)}")

    def _ensure(self, model: DeviceModel):
        import torch
        if self.local_means.shape[0] != model.count:
            self.local_means = torch.zeros((model.count, 3), dtype=torch.float64, device=self._dev)
            self.local_rotations = torch.tensor([1.0, 0, 0, 0], dtype=torch.float64,
                                                device=self._dev).repeat(model.count, 1)

    def refresh_locals(self, model: DeviceModel, rows=None):
        """Re-derive the local poses of the dynamic rows in `rows` (default:
        every row) from their current world pose (ref model.py:371-387)."""
        import torch
        self._ensure(model)
        c = _lib.ctx(model.device.index)
        c.bind_stream()
        if rows is None:
            ids = torch.unique(model.object_ids)
            rt = None
        else:
            rt = torch.as_tensor(np.asarray(rows, np.int64), device=model.device)
            ids = torch.unique(model.object_ids[rt]) if rt.numel() else torch.zeros(0, dtype=torch.int32)
        for oid in ids.cpu().tolist():
            if oid == 0:
                continue
            q, t = self.get_transform(int(oid))
            qa, ta = (_lib.f64 * 4)(*q), (_lib.f64 * 3)(*t)
            if rt is None:
                c.check(c.lib.ss_refresh_object_locals(c.handle, model.struct(), int(oid), 0,
                                                       _lib.ptr(self.local_means), _lib.ptr(self.local_rotations),
                                                       qa, ta))
            else:
                c.check(c.lib.ss_refresh_object_locals_rows(c.handle, model.struct(), int(oid), _lib.ptr(rt),
                                                            int(rt.numel()), _lib.ptr(self.local_means),
                                                            _lib.ptr(self.local_rotations), qa, ta))

    def apply_transform(self, model: DeviceModel, object_id: int, quat, translation, return_rows: bool = True):
        """Set a new transform and rewrite the object's world rows; returns the
        moved rows (ref model.py:389-404), or None with return_rows=False (no
        host read-back: a 60 Hz tick's path)."""
        import torch
        object_id = int(object_id)
        if object_id not in self.transforms:
            raise KeyError(f"unknown object_id {object_id}")
        self.set_transform(object_id, quat, translation)
        self._ensure(model)
        q, t = self.transforms[object_id]
        if not return_rows:
            c = _lib.ctx(model.device.index)
            c.bind_stream()
            c.check(c.lib.ss_apply_object_transform(c.handle, model.struct(), object_id, _lib.ptr(self.local_means),
                                                    _lib.ptr(self.local_rotations), (_lib.f64 * 4)(*q),
                                                    (_lib.f64 * 3)(*t)))
            return None
        rows = torch.nonzero(model.object_ids == object_id).reshape(-1)
        if rows.numel():
            c = _lib.ctx(model.device.index)
            c.bind_stream()
            c.check(c.lib.ss_apply_object_transform(c.handle, model.struct(), object_id, _lib.ptr(self.local_means),
                                                    _lib.ptr(self.local_rotations), (_lib.f64 * 4)(*q),
                                                    (_lib.f64 * 3)(*t)))
        return rows.cpu().numpy()


__all__ = ["ObjectRegistry"]
