"""Client-side ingestion on the GPU: drop-in for
ref pkg/src/splatstream/protocol/delta.py:150-303 (decode_delta,
DeltaBaselines, advance_baseline, apply_delta) and protocol/snapshot.py:85-168
(decode_snapshot), with the replica and its baselines in HBM.

The host parses headers and runs the compression stage exactly like the
reference (Python's zlib, the same `max_size` bounds) and raises the same
exceptions with the same messages for everything decidable from sizes; the
library (csrc/ss_ingest.cu) validates what needs the block's bytes (varints,
survivor indices, code lengths), reports it in a device status word that is
read back once, and only then applies the block.  Values are bit-identical:
float64 dequantisation, f32(f64(base) + residual) baselines.
"""

from __future__ import annotations

import math
import struct
import zlib
from dataclasses import dataclass
from typing import Optional

import numpy as np

from .. import _lib
from ..errors import ProtocolError
from ..model import DeviceModel

MAX_ROWS = 1 << 24
MODE_DENSE_RESIDUAL, MODE_SPARSE_RESIDUAL, MODE_DENSE_ABSOLUTE = 0, 1, 2
_DHEAD = struct.Struct("<BBBBI")        # delta.py:47
_SHEAD = struct.Struct("<IIBBBB6f")     # snapshot.py:28
# attribute id -> (bits, lo, hi, name) (profiles.py ATTRIBUTE_QUANTIZERS)
_QUANT = {0: (16, None, None, "MEANS"), 1: (8, -10.0, 2.0, "LOG_SCALES"), 2: (10, -1.0, 1.0, "QUATERNIONS"),
          3: (8, -8.0, 8.0, "LOGIT_OPACITIES"), 4: (8, -4.0, 4.0, "SH_DC"), 5: (8, -1.0, 1.0, "SH_REST"),
          6: (1, 0.0, 1.0, "LIGHT_VISIBILITY")}
_RESIDUAL = (0, 1)
_STATUS_ERRORS = {1: ("ValueError", "truncated varint"), 2: ("ValueError", "varint too long"),
                  3: ("ProtocolError", "sparse delta index out of range"), 4: ("ProtocolError", "delta codes truncated")}


def _raise_status(code: int):
    kind, msg = _STATUS_ERRORS[code]
    raise (ValueError if kind == "ValueError" else ProtocolError)(msg)  # the module's ProtocolError at raise time


def packed_size(count: int, bits: int) -> int:
    return (count * bits + 7) // 8


def decompress_block(data: bytes, compression_id: int, max_size: Optional[int] = None) -> bytes:
    """ref protocol/profiles.py:49-68 (host zlib, as in the reference)."""
    if compression_id == 0:
        if max_size is not None and len(data) > max_size:
            raise ProtocolError("block larger than its declared contents")
        return data
    if compression_id == 1:
        try:
            if max_size is None:
                return zlib.decompress(data)
            d = zlib.decompressobj()
            out = d.decompress(data, max_size + 1)
        except zlib.error as e:
            raise ProtocolError(f"corrupt compressed block: {e}") from None
        if len(out) > max_size or d.unconsumed_tail:
            raise ProtocolError("block larger than its declared contents")
        return out
    raise ProtocolError(f"unknown compression id {compression_id}")


def _codes_check(block: bytes, bits: int, count: int):
    """The size checks of _codes_from_bytes (delta.py:56-69)."""
    if bits == 16:
        if len(block) < 2 * count:
            raise ProtocolError("delta codes truncated")
    elif bits == 8:
        if len(block) < count:
            raise ProtocolError("delta codes truncated")
    elif count and len(block) < packed_size(count, bits):
        raise ProtocolError("bit-packed block shorter than declared count")


@dataclass
class _Parsed:
    attr: int
    mode: int
    dims: int
    count: int
    k: int
    bits: int
    lo: float
    hi: float
    block: bytes


def parse_delta(payload: bytes) -> _Parsed:
    """Header + compression stage of decode_delta (delta.py:150-205): every
    check that needs no block contents, in the reference's order."""
    if len(payload) < _DHEAD.size:
        raise ProtocolError("delta payload too short")
    attr, mode, compression_id, dims, count = _DHEAD.unpack_from(payload, 0)
    if attr not in _QUANT:
        raise ProtocolError(f"unknown attribute id {attr}")
    if count > MAX_ROWS:
        raise ProtocolError(f"delta declares {count} rows")
    off = _DHEAD.size
    bits, qlo, qhi, name = _QUANT[attr]
    if mode in (MODE_DENSE_RESIDUAL, MODE_SPARSE_RESIDUAL):
        if attr not in _RESIDUAL:
            raise ProtocolError(f"{name} cannot be residual-coded")
        lo, hi = struct.unpack_from("<ff", payload, off)
        if not (math.isfinite(lo) and math.isfinite(hi)):
            raise ProtocolError("residual range is not finite")
        off += 8
        k = count
        if mode == MODE_SPARSE_RESIDUAL:
            (k,) = struct.unpack_from("<I", payload, off)
            if k > count:
                raise ProtocolError(f"sparse delta touches {k} of {count} rows")
            off += 4
        (blen,) = struct.unpack_from("<I", payload, off)
        off += 4
        block = decompress_block(payload[off:off + blen], compression_id,
                                 max_size=5 * k + packed_size(k * dims, bits))
        if mode == MODE_SPARSE_RESIDUAL:
            if k > len(block):  # decode_varints' up-front check (quantize.py:80-81)
                raise ValueError("truncated varint")
        else:
            _codes_check(block, bits, count * dims)
        return _Parsed(attr, mode, dims, count, k, bits, float(lo), float(hi), block)
    if mode == MODE_DENSE_ABSOLUTE:
        (blen,) = struct.unpack_from("<I", payload, off)
        off += 4
        block = decompress_block(payload[off:off + blen], compression_id, max_size=packed_size(count * dims, bits))
        _codes_check(block, bits, count * dims)
        if qlo is None:
            raise ProtocolError(f"absolute mode not defined for {name}")
        return _Parsed(attr, mode, dims, count, count, bits, qlo, qhi, block)
    raise ProtocolError(f"unknown delta mode {mode}")


_STAGING = {}


def _upload(data: bytes, device):
    """bytes -> device uint8 tensor through a reused pinned staging buffer
    (one host memcpy + one async H2D copy)."""
    import torch
    n = max(len(data), 1)
    key = device.index
    st = _STAGING.get(key)
    if st is None or st[0].numel() < n:
        if st is not None:
            st[1].synchronize()
        st = _STAGING[key] = (torch.empty(max(n, 1 << 20) * 5 // 4, dtype=torch.uint8, pin_memory=True),
                              torch.cuda.Event())
    else:
        st[1].synchronize()  # the previous upload from this buffer has been consumed
    host, ev = st
    if data:
        host.numpy()[:len(data)] = np.frombuffer(data, dtype=np.uint8)
    out = torch.empty(n, dtype=torch.uint8, device=device)
    out.copy_(host[:n], non_blocking=True)
    ev.record(torch.cuda.current_stream(device))
    return out


class _Block:
    """A parsed block on the device plus its status word."""

    def __init__(self, p: _Parsed, device):
        import torch
        self.p = p
        self.device = device
        self.data = _upload(p.block, device)
        self.status = torch.zeros(2, dtype=torch.int64, device=device)  # ss_ingest_status (16 B)
        self.indices = torch.empty(max(p.k if p.mode == MODE_SPARSE_RESIDUAL else 0, 1), dtype=torch.int64,
                                   device=device)

    def struct(self, baseline=None, target=None, row_stride=0, inner=0, outer=0, col0=0) -> _lib.SSDeltaApply:
        p = self.p
        a = _lib.SSDeltaApply()
        a.attribute_id, a.mode, a.dims, a.bits = p.attr, p.mode, p.dims, p.bits
        a.count, a.k = p.count, p.k
        a.lo, a.hi = p.lo, p.hi
        a.block, a.block_len = self.data.data_ptr(), len(p.block)
        a.baseline = _lib.ptr(baseline)
        a.target = _lib.ptr(target)
        a.row_stride = row_stride or p.dims
        a.inner = inner or p.dims
        a.outer, a.col0 = outer, col0
        a.status = self.status.data_ptr()
        return a

    def decode(self, values: bool = False):
        """Validate (and optionally dequantise) on the device; raise like the reference."""
        import torch
        c = _lib.ctx(self.device.index)
        c.bind_stream()
        vals = None
        if values:
            rows = self.p.k if self.p.mode == MODE_SPARSE_RESIDUAL else self.p.count
            vals = torch.empty((rows, self.p.dims), dtype=torch.float64, device=self.device)
        c.check(c.lib.ss_decode_delta(c.handle, self.struct(), _lib.ptr(self.indices), _lib.ptr(vals)))
        code = int(self.status[0].item())
        if code:
            _raise_status(code)
        return vals


@dataclass
class DeltaUpdate:
    """ref delta.py:139-147."""
    attribute_id: int
    mode: int
    count: int
    dims: int
    indices: Optional[np.ndarray]
    values: np.ndarray


def decode_delta(payload: bytes, device=None) -> DeltaUpdate:
    """ref delta.py:150 -- decoded on the GPU, returned as host arrays."""
    import torch
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    blk = _Block(parse_delta(payload), dev)
    vals = blk.decode(values=True)
    p = blk.p
    idx = blk.indices[:p.k].cpu().numpy() if p.mode == MODE_SPARSE_RESIDUAL else None
    return DeltaUpdate(p.attr, p.mode, p.count, p.dims, idx, vals.cpu().numpy())


@dataclass
class DeviceBaselines:
    """ref delta.py:208-256 (DeltaBaselines) with the mirrors in HBM."""
    means: object = None
    log_scales: object = None
    epoch: int = 0

    def reset_from_model(self, model: DeviceModel, epoch: int):
        self.means = model.means.clone()
        self.log_scales = model.log_scales.clone()
        self.epoch = epoch

    def array_for(self, attribute_id: int):
        if int(attribute_id) == 0:
            return self.means
        if int(attribute_id) == 1:
            return self.log_scales
        raise KeyError(attribute_id)

    def set_array(self, attribute_id: int, values):
        if int(attribute_id) == 0:
            self.means = values
        elif int(attribute_id) == 1:
            self.log_scales = values
        else:
            raise KeyError(attribute_id)


def _reshape_error(size, shape):
    return ValueError(f"cannot reshape array of size {size} into shape {shape}")


def advance_baseline(baseline_rows, indices, values) -> None:
    """ref delta.py:257-266: f32(f64(base) + value) in place, on the device
    (numpy arguments are uploaded and the result written back)."""
    import torch
    host = not isinstance(baseline_rows, torch.Tensor)
    dev = torch.device("cuda", torch.cuda.current_device())
    b = torch.from_numpy(np.ascontiguousarray(baseline_rows)).to(dev) if host else baseline_rows
    v = values if isinstance(values, torch.Tensor) else torch.from_numpy(np.asarray(values, np.float64))
    v = v.to(b.device, torch.float64)
    flat = b.reshape(b.shape[0], -1)
    if indices is None:
        flat.copy_((flat.double() + v.reshape(flat.shape)).to(flat.dtype))
    else:
        idx = torch.as_tensor(np.asarray(indices, np.int64), device=b.device)
        flat[idx] = (flat[idx].double() + v.reshape(-1, flat.shape[1])).to(flat.dtype)
    if host:
        baseline_rows[...] = b.cpu().numpy().reshape(baseline_rows.shape)


def _apply_delta_host(model, baselines, payload, frame_epoch, current_epoch) -> bool:
    """apply_delta for a host replica (the reference's numpy GaussianModel and
    DeltaBaselines): uploaded, applied on the device, the touched arrays
    written back in place -- as the reference mutates them."""
    import torch
    dm = DeviceModel.from_host(model)
    dev = dm.device
    up = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(dev).reshape(-1, 3)
    db = DeviceBaselines(up(baselines.means), up(baselines.log_scales), getattr(baselines, "epoch", 0))
    ok = apply_delta(dm, db, payload, frame_epoch, current_epoch)
    if not ok:
        return False
    a = model.active_count
    attr = payload[0]
    if attr in _RESIDUAL:
        name = "means" if attr == 0 else "log_scales"
        base = baselines.array_for(attr)
        base[:a] = db.array_for(attr)[:a].cpu().numpy().astype(base.dtype, copy=False).reshape(base[:a].shape)
        getattr(model, name)[:a] = base[:a]
    else:
        name = {2: "quaternions", 3: "logit_opacities", 4: "sh_coeffs", 5: "sh_coeffs", 6: "light_visibility"}[attr]
        dst = getattr(model, name)
        dst[:a] = getattr(dm, name)[:a].cpu().numpy().astype(dst.dtype, copy=False).reshape(dst[:a].shape)
    return True


def apply_delta(model: DeviceModel, baselines: DeviceBaselines, payload: bytes, frame_epoch: int,
                current_epoch: int) -> bool:
    """ref delta.py:269-303 on a device replica: False (untouched) on an epoch
    mismatch; the same exceptions as the reference for malformed payloads,
    raised before anything is written.  A host replica (numpy model and
    baselines) is applied through the device and written back in place."""
    if frame_epoch != current_epoch:
        return False
    if not isinstance(model, DeviceModel):
        return _apply_delta_host(model, baselines, payload, frame_epoch, current_epoch)
    blk = _Block(parse_delta(payload), model.device)
    blk.decode()
    p = blk.p
    a = model.active_count
    if p.count != a:
        raise ProtocolError(f"delta covers {p.count} rows, active is {a}")
    B = (model.sh_degree + 1) ** 2
    if p.attr in _RESIDUAL:
        base = baselines.array_for(p.attr)
        target = model.means if p.attr == 0 else model.log_scales
        if p.dims != 3:
            raise _reshape_error(a * p.dims, (a, 3))
        s = blk.struct(base, target, 3)
    elif p.attr == 2:
        if p.dims != 4:
            raise _reshape_error(a * p.dims, (a, 4))
        s = blk.struct(None, model.quaternions, 4)
    elif p.attr == 3:
        if p.dims != 1:
            raise _reshape_error(a * p.dims, (a,))
        s = blk.struct(None, model.logit_opacities, 1)
    elif p.attr == 4:
        if p.dims != 3:
            raise _reshape_error(a * p.dims, (a, 3))
        s = blk.struct(None, model.sh_coeffs, 3 * B, 1, B, 0)
    elif p.attr == 5:
        if p.dims != 3 * (B - 1):
            raise ProtocolError("sh_rest dims mismatch")
        s = blk.struct(None, model.sh_coeffs, 3 * B, B - 1, B, 1)
    else:
        if p.dims != 1:
            raise _reshape_error(a * p.dims, (a,))
        s = blk.struct(None, model.light_visibility, 1)
    c = _lib.ctx(model.device.index)
    c.bind_stream()
    c.check(c.lib.ss_apply_delta(c.handle, s, _lib.ptr(blk.indices)))
    return True


def decode_snapshot(payload: bytes, device=None):
    """ref snapshot.py:85-168 -- returns (DeviceModel, info)."""
    import torch
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    if len(payload) < _SHEAD.size + 4:
        raise ProtocolError("snapshot payload too short")
    n, active, degree, profile_id, compression_id, _, *aabb = _SHEAD.unpack_from(payload, 0)
    (block_len,) = struct.unpack_from("<I", payload, _SHEAD.size)
    start = _SHEAD.size + 4
    if len(payload) < start + block_len:
        raise ProtocolError("snapshot block truncated")
    if not 0 <= active <= n:
        raise ProtocolError(f"active count {active} exceeds row count {n}")
    if degree > 3:
        raise ProtocolError(f"unsupported sh degree {degree}")
    if n > MAX_ROWS:
        raise ProtocolError(f"snapshot declares {n} rows")
    B = (degree + 1) ** 2
    if profile_id == 1:
        expected = (52 + 12 * B) * n
    elif profile_id == 0:
        expected = (13 + 3 * (B - 1)) * n + packed_size(4 * n, 10) + packed_size(n, 1) + 5 * n
    else:
        raise ProtocolError(f"unknown profile id {profile_id}")
    data = decompress_block(payload[start:start + block_len], compression_id, max_size=expected)
    lo = np.asarray(aabb[:3], dtype=np.float64)
    hi = np.asarray(aabb[3:], dtype=np.float64)
    if not (np.isfinite(lo).all() and np.isfinite(hi).all()):
        raise ProtocolError("snapshot bounds are not finite")
    if profile_id == 1:
        sections = (("means", 12 * n), ("log_scales", 12 * n), ("quaternions", 16 * n), ("opacities", 4 * n),
                    ("sh", 12 * B * n), ("visibility", 4 * n), ("object_ids", 4 * n))
    else:
        sections = [("means", 6 * n), ("log_scales", 3 * n), ("quaternions", packed_size(4 * n, 10)),
                    ("opacities", n), ("sh_dc", 3 * n)]
        if B > 1:
            sections.append(("sh_rest", 3 * (B - 1) * n))
        sections.append(("visibility", packed_size(n, 1)))
    off = 0
    for what, nbytes in sections:
        if off + nbytes > len(data):
            raise ProtocolError(f"snapshot {what} section truncated")
        off += nbytes
    if profile_id == 0 and n > len(data) - off:  # decode_varints' up-front check
        raise ValueError("truncated varint")

    m = DeviceModel(torch.empty((n, 3), dtype=torch.float32, device=dev),
                    torch.empty((n, 3), dtype=torch.float32, device=dev),
                    torch.empty((n, 4), dtype=torch.float32, device=dev),
                    torch.empty(n, dtype=torch.float32, device=dev),
                    (torch.zeros if profile_id == 0 else torch.empty)((n, 3, B), dtype=torch.float32, device=dev),
                    torch.empty(n, dtype=torch.float32, device=dev),
                    torch.empty(n, dtype=torch.int32, device=dev), int(active), int(degree))
    if n:
        blk = _upload(data, dev)
        status = torch.zeros(2, dtype=torch.int64, device=dev)
        d = _lib.SSSnapshotDecode()
        d.model = m.struct()
        d.profile_id = profile_id
        d.aabb_lo = _lib.f64arr(lo, 3)
        d.aabb_hi = _lib.f64arr(hi, 3)
        d.block, d.block_len = blk.data_ptr(), len(data)
        d.status = status.data_ptr()
        c = _lib.ctx(dev.index)
        c.bind_stream()
        c.check(c.lib.ss_decode_snapshot(c.handle, d))
        code = int(status[0].item())
        if code:
            _raise_status(code)
    info = {"profile_id": profile_id, "compression_id": compression_id, "aabb_lo": lo, "aabb_hi": hi}
    return m, info


def decode_snapshot_host(payload: bytes, device=None):
    """ref snapshot.py:85 with the reference's return types: (host
    GaussianModel, info), decoded on the device."""
    m, info = decode_snapshot(payload, device)
    return m.to_host(), info


decode_delta_host = decode_delta  # already returns host arrays (ref delta.py:150)

__all__ = ["advance_baseline", "decode_snapshot_host", "decode_delta_host", "DeltaUpdate", "DeviceBaselines", "apply_delta", "decode_delta", "decode_snapshot", "decompress_block",
           "parse_delta", "packed_size"]
