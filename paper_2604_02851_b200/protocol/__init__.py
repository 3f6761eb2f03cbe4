"""Wire encoders on the GPU: drop-in for the hot part of ref
pkg/src/splatstream/protocol/ (delta.py:72 encode_delta, snapshot.py:47
encode_snapshot, packets.py:73 encode_light_visibility).

The payload bytes are produced by bit-exact CUDA kernels (csrc/ss_codec.cu)
in the raw form (compression_id 0).  compression_id 1 runs the reference's
compression stage -- zlib level 6 -- on the host via the library's libz
wrapper, byte-identical to `zlib.compress(block, 6)`.  The `*_device`
variants keep payloads, lengths and baselines in HBM with no host
synchronisation (the throughput path).

The envelope (`frame_bytes`, CRC32) and the constants follow
protocol/framing.py and protocol/profiles.py.  The decode side (client
replica ingestion: decode_delta, apply_delta, decode_snapshot on a device
replica) lives in protocol/ingest.py.
"""

from __future__ import annotations

import ctypes as C
import struct
import zlib
from dataclasses import dataclass
from enum import IntEnum

import numpy as np

from .. import _lib
from ..errors import ProtocolError
from ..model import as_device

MAGIC = b"GS"
MAX_PAYLOAD = 1 << 28
MAX_ROWS = 1 << 24
COMPRESSION_NONE = 0
COMPRESSION_ZLIB = 1


class PacketType(IntEnum):
    OBJECT_ID_MAP = 0x01
    OBJECT_TRANSFORMS = 0x02
    MODEL_SNAPSHOT = 0x03
    TENSOR_METADATA = 0x04
    TENSOR_DELTA = 0x05
    LIGHT_VISIBILITY = 0x06
    GAUSSIAN_ID_ORDERING = 0x07
    LIGHT_STATE = 0x08
    CAMERA_POSE = 0x09


class AttributeId(IntEnum):
    MEANS = 0
    LOG_SCALES = 1
    QUATERNIONS = 2
    LOGIT_OPACITIES = 3
    SH_DC = 4
    SH_REST = 5
    LIGHT_VISIBILITY = 6


@dataclass(frozen=True)
class QuantizationProfile:
    profile_id: int
    compression_id: int = COMPRESSION_ZLIB


PROFILE_DEFAULT = QuantizationProfile(0)
PROFILE_LOSSLESS = QuantizationProfile(1)
ATTRIBUTE_QUANTIZERS = {
    AttributeId.MEANS: (16, None, None),
    AttributeId.LOG_SCALES: (8, -10.0, 2.0),
    AttributeId.QUATERNIONS: (10, -1.0, 1.0),
    AttributeId.LOGIT_OPACITIES: (8, -8.0, 8.0),
    AttributeId.SH_DC: (8, -4.0, 4.0),
    AttributeId.SH_REST: (8, -1.0, 1.0),
    AttributeId.LIGHT_VISIBILITY: (1, 0.0, 1.0),
}
RESIDUAL_ATTRIBUTES = frozenset({AttributeId.MEANS, AttributeId.LOG_SCALES})
DEFAULT_GATING = {AttributeId.MEANS: 1e-3, AttributeId.LOG_SCALES: 1e-3}


def frame_bytes(ptype: int, epoch: int, payload: bytes) -> bytes:
    """ref protocol/framing.py:51-53."""
    body = struct.pack("<BII", int(ptype), epoch, len(payload)) + payload
    return MAGIC + body + struct.pack("<I", zlib.crc32(body))


FRAME_HEAD = 2 + 9  # magic + '<BII' (ptype, epoch, length)
FRAME_TAIL = 4      # '<I' CRC-32 of header + payload
FRAME_OVERHEAD = FRAME_HEAD + FRAME_TAIL


def crc32_combine(crc1: int, crc2: int, len2: int) -> int:
    """zlib.crc32(A + B) from crc32(A), crc32(B) and len(B) (host arithmetic
    in the library, no data access)."""
    return int(_lib.load_library().ss_crc32_combine(crc1 & 0xFFFFFFFF, crc2 & 0xFFFFFFFF, int(len2)))


def crc32_device(data, length=None):
    """zlib.crc32 of a device uint8 tensor's first `length` bytes (an int, or
    a device int64 scalar tensor such as PayloadBuffer.length; default: all),
    computed on the GPU; returns a device int32 tensor (the CRC's bits)."""
    import torch
    c = _lib.ctx(data.device.index)
    c.bind_stream()
    out = torch.empty(1, dtype=torch.int32, device=data.device)
    n = data.numel()
    if isinstance(length, int):
        n, length = min(n, length), None
    c.check(c.lib.ss_crc32(c.handle, data.data_ptr(), length.data_ptr() if length is not None else None, n,
                           out.data_ptr()))
    return out


def host_zlib(block: bytes) -> bytes:
    """The compression stage through the library's libz (compress2, level 6).
    No Python-side copies; ctypes releases the GIL for the call, so blocks
    compress in parallel from threads (see compress_blocks)."""
    lib = _lib.load_library()
    block = bytes(block)
    n = len(block)
    cap = int(lib.ss_host_zlib_bound(n))
    dst = C.create_string_buffer(cap)
    out = _lib.u64(0)
    src = C.c_char_p(block) if n else C.c_char_p(b"\0")
    if lib.ss_host_zlib_compress(C.cast(src, C.c_void_p), n, C.cast(dst, C.c_void_p), cap, C.byref(out)) != 0:
        raise RuntimeError("zlib compress2 failed")
    return C.string_at(dst, out.value)


_POOL = None


def compress_blocks(blocks):
    """host_zlib of several independent blocks on parallel host threads
    (SURVEY §8f rank 3): every block is one deflate stream, so the bytes are
    those of the serial reference (protocol/profiles.py:41-46)."""
    global _POOL
    blocks = list(blocks)
    if len(blocks) <= 1:
        return [host_zlib(b) for b in blocks]
    if _POOL is None:
        import os
        from concurrent.futures import ThreadPoolExecutor
        _POOL = ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 4))
    return list(_POOL.map(host_zlib, blocks))


def _recompress_delta(raw: bytes, compression_id: int) -> bytes:
    if compression_id == COMPRESSION_NONE:
        return raw
    if compression_id != COMPRESSION_ZLIB:
        raise ProtocolError(f"unknown compression id {compression_id}")
    mode = raw[1]
    head = 8 + (12 if mode == 1 else 8 if mode == 0 else 0)
    (blen,) = struct.unpack_from("<I", raw, head)
    block = host_zlib(raw[head + 4: head + 4 + blen])
    hdr = bytearray(raw[:head])
    hdr[2] = COMPRESSION_ZLIB
    return bytes(hdr) + struct.pack("<I", len(block)) + block


def _recompress_deltas(raws, compression_id: int):
    """_recompress_delta of several payloads, their blocks deflated in parallel."""
    if compression_id == COMPRESSION_NONE:
        return list(raws)
    if compression_id != COMPRESSION_ZLIB:
        raise ProtocolError(f"unknown compression id {compression_id}")
    heads, blocks = [], []
    for raw in raws:
        mode = raw[1]
        head = 8 + (12 if mode == 1 else 8 if mode == 0 else 0)
        (blen,) = struct.unpack_from("<I", raw, head)
        hdr = bytearray(raw[:head])
        hdr[2] = COMPRESSION_ZLIB
        heads.append(bytes(hdr))
        blocks.append(raw[head + 4: head + 4 + blen])
    return [h + struct.pack("<I", len(b)) + b for h, b in zip(heads, compress_blocks(blocks))]


def _recompress_snapshot(raw: bytes, compression_id: int) -> bytes:
    if compression_id == COMPRESSION_NONE:
        return raw
    if compression_id != COMPRESSION_ZLIB:
        raise ProtocolError(f"unknown compression id {compression_id}")
    (blen,) = struct.unpack_from("<I", raw, 36)
    block = host_zlib(raw[40:40 + blen])
    hdr = bytearray(raw[:36])
    hdr[10] = COMPRESSION_ZLIB
    return bytes(hdr) + struct.pack("<I", len(block)) + block


class PayloadBuffer:
    """Device output buffer + device length word, reused across calls."""

    def __init__(self, capacity: int, device):
        import torch
        self.data = torch.empty(max(int(capacity), 64), dtype=torch.uint8, device=device)
        self.length = torch.zeros(1, dtype=torch.int64, device=device)

    def ensure(self, capacity: int):
        import torch
        if self.data.numel() < capacity:
            self.data = torch.empty(int(capacity * 1.25) + 64, dtype=torch.uint8, device=self.data.device)

    def to_bytes(self) -> bytes:
        n = int(self.length.item())
        return self.data[:n].cpu().numpy().tobytes()


def _dims_of(shape):
    return 1 if len(shape) == 1 else int(np.prod(shape[1:]))


def encode_delta_device(attribute_id, current, baseline=None, new_baseline=None, gating_threshold=None,
                        out: PayloadBuffer = None):
    """Raw (compression 0) delta payload into `out` (device), no host sync.
    current/baseline: torch CUDA float32/float64 tensors, (rows, ...)."""
    import torch
    attr = AttributeId(attribute_id)
    rows = int(current.shape[0])
    dims = _dims_of(tuple(current.shape))
    c = _lib.ctx(current.device.index)
    cur = current.contiguous()
    dt = 1 if cur.dtype == torch.float64 else 0
    if cur.dtype not in (torch.float32, torch.float64):
        cur = cur.float()
        dt = 0
    base = None
    if attr in RESIDUAL_ATTRIBUTES:
        if baseline is None:
            raise ValueError(f"{attr.name} is residual-coded and needs a baseline")
        if tuple(baseline.shape[:1]) != (rows,) or _dims_of(tuple(baseline.shape)) != dims:
            raise ValueError("baseline shape mismatch")
        base = baseline.contiguous().to(cur.dtype)
    gate = DEFAULT_GATING.get(attr, 0.0) if gating_threshold is None else float(gating_threshold)
    bound = int(c.lib.ss_delta_bound(int(attr), rows, dims))
    if out is None:
        out = PayloadBuffer(bound, current.device)
    out.ensure(bound)
    c.check(c.lib.ss_encode_delta(c.handle, int(attr), _lib.ptr(cur), dt, _lib.ptr(base), _lib.ptr(new_baseline),
                                  rows, dims, gate, _lib.ptr(out.data), out.data.numel(), _lib.ptr(out.length)))
    return out


class DeltaTicker:
    """One server tick's deltas for a DeviceModel in ONE library call
    (one kernel launch, no host sync): attributes in emission order (ref
    server.py:67-74, 488-493), residual baselines advanced in place, payloads
    into `outs[attr]` (PayloadBuffer).  SH DC / SH rest are read in place from
    the (N, 3, B) coefficients.  The ctypes job array is built once per set of
    attributes, so a 60 Hz loop pays one foreign call per tick."""

    def __init__(self, model, baselines, outs, gating=None):
        self.model, self.baselines, self.outs, self.gating = model, baselines, outs, gating
        self._jobs = {}
        self._ctx = _lib.ctx(model.device.index)

    def _build(self, attributes):
        model = self.model
        a = model.active_count
        B = (model.sh_degree + 1) ** 2
        jobs = (_lib.SSDeltaJob * len(attributes))()
        for i, attr in enumerate(attributes):
            attr = AttributeId(attr)
            j = jobs[i]
            j.attribute_id = int(attr)
            j.in_dtype = 0
            j.rows = a
            j.gating_threshold = DEFAULT_GATING.get(attr, 0.0) if self.gating is None else float(self.gating)
            if attr == AttributeId.MEANS or attr == AttributeId.LOG_SCALES:
                src = model.means if attr == AttributeId.MEANS else model.log_scales
                base = self.baselines[int(attr)]
                j.cur, j.base, j.new_base, j.dims = src.data_ptr(), base.data_ptr(), base.data_ptr(), 3
            elif attr == AttributeId.QUATERNIONS:
                j.cur, j.dims = model.quaternions.data_ptr(), 4
            elif attr == AttributeId.LOGIT_OPACITIES:
                j.cur, j.dims = model.logit_opacities.data_ptr(), 1
            elif attr == AttributeId.SH_DC:
                j.cur, j.dims, j.row_stride, j.inner, j.outer, j.col0 = model.sh_coeffs.data_ptr(), 3, 3 * B, 1, B, 0
            elif attr == AttributeId.SH_REST:
                if B == 1:
                    raise ValueError("sh_rest needs sh_degree > 0")
                j.cur, j.dims, j.row_stride, j.inner, j.outer, j.col0 = (model.sh_coeffs.data_ptr(), 3 * (B - 1),
                                                                         3 * B, B - 1, B, 1)
            else:
                j.cur, j.dims = model.light_visibility.data_ptr(), 1
            buf = self.outs[int(attr)]
            buf.ensure(int(self._ctx.lib.ss_delta_bound(int(attr), a, j.dims)))
            j.out, j.out_cap, j.out_len = buf.data.data_ptr(), buf.data.numel(), buf.length.data_ptr()
        return jobs

    def _key(self, attributes):
        m = self.model
        ptrs = tuple(t.data_ptr() for t in (m.means, m.log_scales, m.quaternions, m.logit_opacities, m.sh_coeffs,
                                            m.light_visibility))
        bptrs = tuple(int(b.data_ptr()) for b in self.baselines.values())
        # the output buffers too: PayloadBuffer.ensure() may reallocate one, and
        # a cached job array must never point at a freed payload buffer
        optrs = tuple(int(self.outs[int(x)].data.data_ptr()) for x in attributes)
        return tuple(int(x) for x in attributes), m.active_count, ptrs, bptrs, optrs

    def __call__(self, attributes):
        # the job array is rebuilt when the active prefix or a buffer changes
        full = self._key(attributes)
        key = full[0]
        jobs = self._jobs.get(full)
        if jobs is None:
            if len(self._jobs) > 32:
                self._jobs.clear()
            jobs = self._build(key)  # may grow (reallocate) output buffers:
            full = self._key(attributes)  # key the jobs by the pointers they hold
            self._jobs[full] = jobs
        import torch
        done = getattr(self, "_read_done", None)
        if done is not None:  # the last read_async's copies of the output buffers (side stream)
            torch.cuda.current_stream(self.model.device).wait_event(done)
            self._read_done = None
        c = self._ctx
        c.bind_stream()
        c.check(c.lib.ss_encode_delta_batch(c.handle, jobs, len(key)))
        return self.model.active_count * len(key)

    def read_async(self, attributes, frame_epoch=None):
        """Start reading the last call's payloads for `attributes` back without
        a host sync: lengths and each payload's bound-sized buffer are copied
        into pinned memory on a side stream (after the encode; the next
        encode waits for the copies), so the work queued after this call --
        the next optimizer step -- runs while the payloads cross PCIe;
        `.result()` waits for that copy only.

        With `frame_epoch`, `.result()` returns TENSOR_DELTA frames instead
        (ref framing.py:51-53): each payload lands in pinned memory between
        its envelope header and CRC, and the CRC of the payload is computed on
        the device (ss_crc32), so the host never reads the payload bytes."""
        import torch
        key = [int(x) for x in attributes]
        m = self.model
        frames = frame_epoch is not None
        pad = FRAME_OVERHEAD if frames else 0
        bounds = [int(self._ctx.lib.ss_delta_bound(a, m.active_count, self._dims(a))) + pad for a in key]
        need = sum(bounds)
        slot = getattr(self, "_slot", 0) ^ 1  # two pinned buffers: one may still be pending
        self._slot = slot
        bufs = getattr(self, "_async", None)
        if bufs is None:
            bufs = self._async = [None, None]
        st = bufs[slot]
        if st is not None:
            st[2].synchronize()  # its previous reader has finished with it
        if st is None or st[0].numel() < need:
            st = bufs[slot] = (torch.empty(max(need, 1 << 16) * 5 // 4, dtype=torch.uint8, pin_memory=True),
                               torch.empty(8, dtype=torch.int64, pin_memory=True), torch.cuda.Event(),
                               torch.empty(8, dtype=torch.int32, pin_memory=True))
        host, lens, ev, crcs = st
        if frames:
            dcrc = getattr(self, "_dcrc", None)
            if dcrc is None:
                dcrc = self._dcrc = torch.empty(8, dtype=torch.int32, device=m.device)
            c = self._ctx
            c.bind_stream()
        cur = torch.cuda.current_stream(m.device)
        last = getattr(self, "_read_last", None)
        if last is not None:  # the previous copies out of dcrc / the payload buffers are done
            cur.wait_event(last)
        if frames:
            for i, (a, b) in enumerate(zip(key, bounds)):
                out = self.outs[a]
                c.check(c.lib.ss_crc32(c.handle, out.data.data_ptr(), out.length.data_ptr(), b - pad,
                                       dcrc[i:].data_ptr()))
        cs = getattr(self, "_copy_stream", None)
        if cs is None:
            cs = self._copy_stream = torch.cuda.Stream(m.device)
        cs.wait_stream(cur)
        off = 0
        with torch.cuda.stream(cs):
            for i, (a, b) in enumerate(zip(key, bounds)):
                out = self.outs[a]
                # payload bytes between the frame's header and CRC slots
                host[off + (FRAME_HEAD if frames else 0):off + b - (FRAME_TAIL if frames else 0)].copy_(
                    out.data[:b - pad], non_blocking=True)
                lens[i:i + 1].copy_(out.length, non_blocking=True)
                off += b
            if frames:
                crcs[:len(key)].copy_(dcrc[:len(key)], non_blocking=True)
        ev.record(cs)
        self._read_done = self._read_last = ev
        return _PendingPayloads(host, lens, ev, bounds, crcs if frames else None, frame_epoch)

    def _dims(self, attr):
        m = self.model
        B = (m.sh_degree + 1) ** 2
        return {0: 3, 1: 3, 2: 4, 3: 1, 4: 3, 5: 3 * (B - 1), 6: 1}[int(attr)]

    def read(self, attributes, copy: bool = True):
        """Payloads of the last call for `attributes`, read back with two host
        syncs in total (lengths, then every payload into pinned memory).
        copy=False returns memoryviews of that pinned buffer (no host-side
        copy; valid until the next read)."""
        import torch
        key = [int(x) for x in attributes]
        if not key:
            return []
        lens = torch.cat([self.outs[a].length for a in key]).cpu().tolist()
        total = int(sum(lens))
        host = getattr(self, "_pinned", None)
        if host is None or host.numel() < total:
            host = self._pinned = torch.empty(max(total, 1 << 16) * 5 // 4, dtype=torch.uint8, pin_memory=True)
        off = 0
        for a, n in zip(key, lens):
            host[off:off + n].copy_(self.outs[a].data[:n], non_blocking=True)
            off += n
        torch.cuda.current_stream(self.model.device).synchronize()
        mv = memoryview(host.numpy())
        out, off = [], 0
        for n in lens:
            out.append(mv[off:off + n].tobytes() if copy else mv[off:off + n])
            off += n
        return out


class _PendingPayloads:
    """Payload bytes (or frames) of one tick, copied back asynchronously
    (DeltaTicker.read_async)."""

    def __init__(self, host, lens, ev, bounds, crcs=None, epoch=None):
        self.host, self.lens, self.ev, self.bounds, self.crcs, self.epoch = host, lens, ev, bounds, crcs, epoch

    def result(self, copy: bool = True):
        self.ev.synchronize()
        hv = self.host.numpy()
        mv = memoryview(hv)
        ln = self.lens.numpy()
        out, off = [], 0
        for i, b in enumerate(self.bounds):
            n = int(ln[i])
            if self.crcs is None:
                out.append(mv[off:off + n].tobytes() if copy else mv[off:off + n])
            else:
                head = struct.pack("<BII", int(PacketType.TENSOR_DELTA), self.epoch, n)
                crc = crc32_combine(zlib.crc32(head), int(self.crcs[i]) & 0xFFFFFFFF, n)
                hv[off:off + FRAME_HEAD] = np.frombuffer(MAGIC + head, np.uint8)
                hv[off + FRAME_HEAD + n:off + FRAME_HEAD + n + FRAME_TAIL] = np.frombuffer(struct.pack("<I", crc), np.uint8)
                k = FRAME_HEAD + n + FRAME_TAIL
                out.append(mv[off:off + k].tobytes() if copy else mv[off:off + k])
            off += b
        return out


# ref server.py:57-74: per-attribute periods (ticks) and the fixed emission order
DEFAULT_DELTA_PERIODS = {AttributeId.LOGIT_OPACITIES: 1, AttributeId.SH_DC: 1, AttributeId.MEANS: 1,
                         AttributeId.LOG_SCALES: 1, AttributeId.QUATERNIONS: 10, AttributeId.SH_REST: 30}
DELTA_ORDER = (AttributeId.MEANS, AttributeId.LOG_SCALES, AttributeId.QUATERNIONS, AttributeId.LOGIT_OPACITIES,
               AttributeId.SH_DC, AttributeId.SH_REST)


def due_attributes(tick_index: int, periods=None, appended: bool = False, sh_degree: int = 3):
    """Attributes StreamServer emits at `tick_index`, in emission order (ref
    server.py:89-91 DeltaSchedule.due, 488-493; SH rest is skipped at degree
    0, server.py:352-354)."""
    periods = DEFAULT_DELTA_PERIODS if periods is None else periods
    out = []
    for attr in DELTA_ORDER:
        p = periods.get(attr)
        if appended or (p is not None and tick_index % p == 0):
            if attr == AttributeId.SH_REST and sh_degree == 0:
                continue
            out.append(attr)
    return out


class DeltaEmitter:
    """StreamServer's per-tick delta emission (ref server.py:336-358 +
    488-493) on a DeviceModel: the due attributes encoded in one batched
    library call, residual baselines (rows [:a] of the server's
    DeviceBaselines) advanced in HBM, payloads read back and passed through
    the compression stage -- byte-identical to the reference server's
    TENSOR_DELTA payloads."""

    def __init__(self, model, baselines, compression_id: int = COMPRESSION_ZLIB, periods=None):
        self.model, self.baselines, self.compression_id, self.periods = model, baselines, compression_id, periods
        self._outs = {int(a): PayloadBuffer(1 << 16, model.device) for a in AttributeId}
        self._ticker = None
        self._state = None

    def tick(self, tick_index: int, appended: bool = False):
        """[(attribute_id, payload bytes)] for the attributes due at this tick."""
        m = self.model
        a = m.active_count
        if a == 0:  # server.py:491: no deltas without active rows
            return []
        due = [int(x) for x in due_attributes(tick_index, self.periods, appended, m.sh_degree)]
        if not due:
            return []
        state = (a, self.baselines.means.data_ptr(), self.baselines.log_scales.data_ptr())
        if self._ticker is None or self._state != state:  # new active prefix or baselines (snapshot reset)
            self._ticker = DeltaTicker(m, {0: self.baselines.means[:a], 1: self.baselines.log_scales[:a]}, self._outs)
            self._state = state
        self._ticker(due)
        raw = self._ticker.read(due)
        if self.compression_id == COMPRESSION_NONE:
            return list(zip(due, raw))
        return list(zip(due, _recompress_deltas(raw, self.compression_id)))


def delta_tick_device(model, attributes, baselines, outs, gating=None):
    """One-shot DeltaTicker call (see DeltaTicker)."""
    return DeltaTicker(model, baselines, outs, gating)(attributes)


def encode_delta(attribute_id, current, baseline=None, gating_threshold=None, compression_id: int = COMPRESSION_ZLIB):
    """ref protocol/delta.py:72 -- returns (payload bytes, new baseline or None).

    Host arrays are uploaded; float32 and float64 inputs are both encoded
    exactly (a float64 residual of float32 values is computed in float64 either
    way).  For CUDA tensor inputs the new baseline is returned as a tensor."""
    import torch
    attr = AttributeId(attribute_id)
    dev = current.device if isinstance(current, torch.Tensor) and current.is_cuda else \
        torch.device("cuda", torch.cuda.current_device())

    def to_dev(x):
        if isinstance(x, torch.Tensor):
            return x.to(dev)
        a = np.asarray(x)
        return torch.from_numpy(np.ascontiguousarray(a, np.float32 if a.dtype == np.float32 else np.float64)).to(dev)

    cur = to_dev(current)
    base = new_base = None
    if attr in RESIDUAL_ATTRIBUTES:
        if baseline is None:
            raise ValueError(f"{attr.name} is residual-coded and needs a baseline")
        base = to_dev(baseline)
        if base.shape[0] != cur.shape[0] or base.numel() != cur.numel():
            raise ValueError("baseline shape mismatch")
        if torch.float64 in (cur.dtype, base.dtype):
            cur, base = cur.double(), base.double()
        new_base = torch.empty(tuple(base.shape), dtype=torch.float32, device=dev)
    out = encode_delta_device(attr, cur, base, new_base, gating_threshold)
    payload = _recompress_delta(out.to_bytes(), compression_id)
    if new_base is None:
        return payload, None
    if isinstance(baseline, torch.Tensor):
        return payload, new_base
    return payload, new_base.cpu().numpy().reshape(np.asarray(baseline).shape)


def encode_snapshot_device(model, profile_id: int, out: PayloadBuffer = None, base_means=None, base_log_scales=None):
    """Raw snapshot payload into `out` (device) plus the decoded means/log
    scales (server baseline reset, ref server.py:481-484), no host sync."""
    dm, _ = as_device(model)
    c = _lib.ctx(dm.device.index)
    bound = int(c.lib.ss_snapshot_bound(dm.count, dm.sh_degree, int(profile_id)))
    if out is None:
        out = PayloadBuffer(bound, dm.device)
    out.ensure(bound)
    c.check(c.lib.ss_encode_snapshot(c.handle, dm.struct(), int(profile_id), _lib.ptr(out.data), out.data.numel(),
                                     _lib.ptr(out.length), _lib.ptr(base_means), _lib.ptr(base_log_scales)))
    return out


def encode_snapshot(model, profile: QuantizationProfile = PROFILE_DEFAULT, return_baselines: bool = False):
    """ref protocol/snapshot.py:47 -- payload bytes [, (base_means, base_log_scales)]."""
    import torch
    dm, _ = as_device(model)
    bm = torch.empty((dm.count, 3), dtype=torch.float32, device=dm.device) if return_baselines else None
    bl = torch.empty((dm.count, 3), dtype=torch.float32, device=dm.device) if return_baselines else None
    out = encode_snapshot_device(dm, profile.profile_id, None, bm, bl)
    payload = _recompress_snapshot(out.to_bytes(), profile.compression_id)
    if return_baselines:
        return payload, (bm.cpu().numpy(), bl.cpu().numpy())
    return payload


def encode_light_visibility_device(visibility, out: PayloadBuffer = None) -> PayloadBuffer:
    """ref protocol/packets.py:73-76 into a device PayloadBuffer (no host sync)."""
    import torch
    if isinstance(visibility, torch.Tensor) and visibility.is_cuda:
        v = visibility if visibility.dtype == torch.float32 and visibility.is_contiguous() else \
            visibility.float().contiguous()
    else:
        v = torch.from_numpy(np.ascontiguousarray(np.asarray(visibility), np.float32)).cuda()
    c = _lib.ctx(v.device.index)
    n = v.numel()
    if out is None:
        out = PayloadBuffer(4 + (n + 7) // 8, v.device)
    out.ensure(4 + (n + 7) // 8)
    c.bind_stream()
    c.check(c.lib.ss_encode_light_visibility(c.handle, _lib.ptr(v), n, _lib.ptr(out.data), out.data.numel(),
                                             _lib.ptr(out.length)))
    return out


def encode_light_visibility(visibility) -> bytes:
    """ref protocol/packets.py:73-76."""
    return encode_light_visibility_device(visibility).to_bytes()


# client-side ingestion on the GPU
from .ingest import DeltaUpdate, DeviceBaselines, apply_delta, decode_delta, decode_snapshot  # noqa: E402

__all__ = [n for n in dir() if not n.startswith("_")]
