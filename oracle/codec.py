"""CPU restatement of the splatstream wire encoders (test infrastructure only).

Follows, function by function:
  quantize / dequantize   ref pkg/src/splatstream/protocol/quantize.py:8-24
  pack_lsb                ref protocol/quantize.py:31-38
  leb128                  ref protocol/quantize.py:58-71
  QUANT table, zlib stage ref protocol/profiles.py:28-46
  delta_payload           ref protocol/delta.py:72-137   (encode_delta)
  apply_residual          ref protocol/delta.py:259-266  (advance_baseline)
  snapshot_payload        ref protocol/snapshot.py:47-82 (encode_snapshot)
  snapshot_dequant        ref protocol/snapshot.py:85-168 (decode_snapshot,
                          the part the server uses to reset its baselines,
                          server.py:481-484)
  delta_unpack            ref protocol/delta.py:150-205 (decode_delta)

Everything is vectorised numpy in float64, using only IEEE-exact elementwise
operations, so results are bit-identical to the reference's numpy code and to
the GPU kernels that mirror the same operation order.  Pinned against the
golden vectors in tests/golden (see tests/test_oracle_golden.py).
"""

from __future__ import annotations

import struct
import zlib

import numpy as np

# attribute ids (ref protocol/framing.py:40-47)
MEANS, LOG_SCALES, QUATERNIONS, LOGIT_OPACITIES, SH_DC, SH_REST, LIGHT_VISIBILITY = range(7)

# (bits, lo, hi); means carry their own range (ref protocol/profiles.py:28-36)
QUANT = {
    MEANS: (16, None, None),
    LOG_SCALES: (8, -10.0, 2.0),
    QUATERNIONS: (10, -1.0, 1.0),
    LOGIT_OPACITIES: (8, -8.0, 8.0),
    SH_DC: (8, -4.0, 4.0),
    SH_REST: (8, -1.0, 1.0),
    LIGHT_VISIBILITY: (1, 0.0, 1.0),
}
RESIDUAL = (MEANS, LOG_SCALES)
DEFAULT_GATE = 1e-3  # ref protocol/delta.py:45

MODE_DENSE_RESIDUAL, MODE_SPARSE_RESIDUAL, MODE_DENSE_ABSOLUTE = 0, 1, 2


def quantize(v, lo, hi, bits):
    """rint(clip((clip(v,lo,hi)-lo)/span, 0, 1) * (2^b-1)), span=1 if hi<=lo."""
    v = np.asarray(v, np.float64)
    lo = np.asarray(lo, np.float64)
    hi = np.asarray(hi, np.float64)
    levels = float((1 << bits) - 1)
    span = np.where(hi > lo, hi - lo, 1.0)
    clipped = np.minimum(np.maximum(v, lo), hi)
    t = (clipped - lo) / span
    t = np.minimum(np.maximum(t, 0.0), 1.0)
    return np.rint(t * levels).astype(np.uint32)


def dequantize(codes, lo, hi, bits):
    levels = float((1 << bits) - 1)
    lo = np.asarray(lo, np.float64)
    hi = np.asarray(hi, np.float64)
    return lo + (np.asarray(codes, np.float64) / levels) * (hi - lo)


def pack_lsb(codes, bits) -> bytes:
    """Concatenate `bits`-wide codes into one little-endian bit stream."""
    c = np.asarray(codes, np.uint64).ravel()
    if c.size == 0:
        return b""
    planes = (c[:, None] >> np.arange(bits, dtype=np.uint64)[None, :]) & np.uint64(1)
    return np.packbits(planes.astype(np.uint8).ravel(), bitorder="little").tobytes()


def unpack_lsb(data: bytes, bits, count):
    if count == 0:
        return np.zeros(0, np.uint32)
    raw = np.frombuffer(data[: (count * bits + 7) // 8], np.uint8)
    stream = np.unpackbits(raw, bitorder="little")[: count * bits].reshape(count, bits)
    w = (np.uint64(1) << np.arange(bits, dtype=np.uint64))
    return (stream.astype(np.uint64) * w).sum(axis=1).astype(np.uint32)


def leb128(values) -> bytes:
    """Unsigned LEB128 of every value, vectorised (no per-value Python loop)."""
    v = np.asarray(values, np.uint64).ravel()
    if v.size == 0:
        return b""
    nbits = np.zeros(v.size, np.int64)
    t = v.copy()
    while t.any():
        nz = t != 0
        nbits[nz] += 1
        t >>= np.uint64(1)
    nbytes = np.maximum(1, (nbits + 6) // 7)
    starts = np.concatenate([[0], np.cumsum(nbytes)[:-1]])
    out = np.zeros(int(nbytes.sum()), np.uint8)
    for j in range(int(nbytes.max())):
        sel = nbytes > j
        chunk = ((v[sel] >> np.uint64(7 * j)) & np.uint64(0x7F)).astype(np.uint8)
        more = (nbytes[sel] - 1 > j).astype(np.uint8) << 7
        out[starts[sel] + j] = chunk | more
    return out.tobytes()


def leb128_decode(data: bytes, count, offset=0):
    vals = np.zeros(count, np.uint64)
    for i in range(count):
        acc, shift = 0, 0
        while True:
            b = data[offset]
            offset += 1
            acc |= (b & 0x7F) << shift
            shift += 7
            if not b & 0x80:
                break
        vals[i] = acc
    return vals, offset


def compress(block: bytes, compression_id: int) -> bytes:
    if compression_id == 0:
        return block
    if compression_id == 1:
        return zlib.compress(block, 6)
    raise ValueError(f"unknown compression id {compression_id}")


def decompress(block: bytes, compression_id: int) -> bytes:
    return block if compression_id == 0 else zlib.decompress(block)


def _code_bytes(codes, bits) -> bytes:
    if bits == 16:
        return np.asarray(codes).astype("<u2").tobytes()
    if bits == 8:
        return np.asarray(codes).astype("<u1").tobytes()
    return pack_lsb(codes, bits)


def _f32_round(x: float) -> float:
    return float(np.float32(x))


def delta_payload(attr, current, baseline=None, gate=None, compression_id=1):
    """Returns (payload bytes, new baseline f32 or None).  ref delta.py:72-137."""
    cur = np.asarray(current, np.float64)
    rows = cur.shape[0]
    dims = 1 if cur.ndim == 1 else int(np.prod(cur.shape[1:]))
    x = cur.reshape(rows, dims)
    bits = QUANT[attr][0]
    if attr in RESIDUAL:
        if baseline is None:
            raise ValueError("residual attribute needs a baseline")
        b = np.asarray(baseline, np.float64).reshape(rows, dims)
        g = DEFAULT_GATE if gate is None else gate
        r = x - b
        row_max = np.abs(r).max(axis=1) if rows else np.zeros(0)
        keep = row_max >= g
        k = int(keep.sum())
        advanced = b.copy()
        if k < 0.5 * rows:
            idx = np.flatnonzero(keep)
            sent = r[idx]
            m = _f32_round(np.abs(sent).max()) if k else 0.0
            codes = quantize(sent, -m, m, bits)
            advanced[idx] = advanced[idx] + dequantize(codes, -m, m, bits)
            prev = np.concatenate([[-1], idx[:-1]]) if k else np.zeros(0, np.int64)
            gaps = idx - prev - 1
            block = leb128(gaps) + _code_bytes(codes, bits)
            mode, extra = MODE_SPARSE_RESIDUAL, struct.pack("<ffI", -m, m, k)
        else:
            m = _f32_round(np.abs(r).max()) if rows else 0.0
            codes = quantize(r, -m, m, bits)
            advanced = advanced + dequantize(codes, -m, m, bits)
            block = _code_bytes(codes, bits)
            mode, extra = MODE_DENSE_RESIDUAL, struct.pack("<ff", -m, m)
        new_base = advanced.astype(np.float32).reshape(np.asarray(baseline).shape)
    else:
        bits, lo, hi = QUANT[attr]
        codes = (x >= 0.5).astype(np.uint32) if attr == LIGHT_VISIBILITY else quantize(x, lo, hi, bits)
        block = _code_bytes(codes, bits)
        mode, extra, new_base = MODE_DENSE_ABSOLUTE, b"", None
    packed = compress(block, compression_id)
    head = struct.pack("<BBBBI", attr, mode, compression_id, dims, rows)
    return head + extra + struct.pack("<I", len(packed)) + packed, new_base


def delta_unpack(payload: bytes):
    """Returns dict(attr, mode, count, dims, indices, values f64)."""
    attr, mode, comp, dims, count = struct.unpack_from("<BBBBI", payload, 0)
    off = 8
    bits = QUANT[attr][0]
    out = dict(attr=attr, mode=mode, count=count, dims=dims, indices=None)
    if mode in (MODE_DENSE_RESIDUAL, MODE_SPARSE_RESIDUAL):
        lo, hi = struct.unpack_from("<ff", payload, off)
        off += 8
        k = count
        if mode == MODE_SPARSE_RESIDUAL:
            (k,) = struct.unpack_from("<I", payload, off)
            off += 4
        (blen,) = struct.unpack_from("<I", payload, off)
        off += 4
        block = decompress(payload[off:off + blen], comp)
        boff = 0
        if mode == MODE_SPARSE_RESIDUAL:
            gaps, boff = leb128_decode(block, k)
            out["indices"] = np.cumsum(gaps.astype(np.int64) + 1) - 1
        codes = _codes_from(block[boff:], bits, k * dims).reshape(k, dims)
        out["values"] = dequantize(codes, lo, hi, bits)
    else:
        (blen,) = struct.unpack_from("<I", payload, off)
        off += 4
        block = decompress(payload[off:off + blen], comp)
        codes = _codes_from(block, bits, count * dims).reshape(count, dims)
        if attr == LIGHT_VISIBILITY:
            out["values"] = codes.astype(np.float64)
        else:
            _, lo, hi = QUANT[attr]
            out["values"] = dequantize(codes, lo, hi, bits)
    return out


def _codes_from(block, bits, n):
    if bits == 16:
        return np.frombuffer(block[:2 * n], "<u2").astype(np.uint32)
    if bits == 8:
        return np.frombuffer(block[:n], "<u1").astype(np.uint32)
    return unpack_lsb(block, bits, n)


def apply_residual(base_rows, indices, values):
    """f32(f64(base) + values), in place.  ref delta.py:259-266."""
    flat = base_rows.reshape(base_rows.shape[0], -1)
    if indices is None:
        flat[:] = (flat.astype(np.float64) + values).astype(np.float32)
    else:
        flat[indices] = (flat[indices].astype(np.float64) + values).astype(np.float32)


def snapshot_payload(means, log_scales, quats, logits, sh, vis, object_ids,
                     active_count, sh_degree, profile_id=0, compression_id=1) -> bytes:
    """ref snapshot.py:47-82."""
    n = means.shape[0]
    if n:
        lo = means.min(axis=0).astype(np.float64)
        hi = means.max(axis=0).astype(np.float64)
    else:
        lo = np.zeros(3)
        hi = np.zeros(3)
    if profile_id == 1:
        sections = [means.astype("<f4"), log_scales.astype("<f4"), quats.astype("<f4"),
                    logits.astype("<f4"), sh.astype("<f4"), vis.astype("<f4"),
                    object_ids.astype("<i4")]
        body = b"".join(s.tobytes() for s in sections)
    elif profile_id == 0:
        parts = [quantize(means, lo, hi, 16).astype("<u2").tobytes()]
        for attr, arr in ((LOG_SCALES, log_scales),):
            b, qlo, qhi = QUANT[attr]
            parts.append(quantize(arr, qlo, qhi, b).astype("<u1").tobytes())
        b, qlo, qhi = QUANT[QUATERNIONS]
        parts.append(pack_lsb(quantize(quats, qlo, qhi, b), b))
        b, qlo, qhi = QUANT[LOGIT_OPACITIES]
        parts.append(quantize(logits, qlo, qhi, b).astype("<u1").tobytes())
        b, qlo, qhi = QUANT[SH_DC]
        parts.append(quantize(sh[:, :, 0], qlo, qhi, b).astype("<u1").tobytes())
        if sh.shape[2] > 1:
            b, qlo, qhi = QUANT[SH_REST]
            parts.append(quantize(sh[:, :, 1:], qlo, qhi, b).astype("<u1").tobytes())
        parts.append(pack_lsb((np.asarray(vis) >= 0.5).astype(np.uint32), 1))
        parts.append(leb128(np.asarray(object_ids).astype(np.int64).astype(np.uint64)))
        body = b"".join(parts)
    else:
        raise ValueError(f"unknown profile id {profile_id}")
    packed = compress(body, compression_id)
    head = struct.pack("<IIBBBB6f", n, active_count, sh_degree, profile_id, compression_id, 0,
                       *lo.astype(np.float32), *hi.astype(np.float32))
    return head + struct.pack("<I", len(packed)) + packed


def snapshot_dequant(payload: bytes):
    """Decode a snapshot to f32 attribute arrays (dict).  ref snapshot.py:85-168."""
    n, active, degree, profile, comp, _, *aabb = struct.unpack_from("<IIBBBB6f", payload, 0)
    (blen,) = struct.unpack_from("<I", payload, 36)
    data = decompress(payload[40:40 + blen], comp)
    B = (degree + 1) ** 2
    lo = np.asarray(aabb[:3], np.float64)
    hi = np.asarray(aabb[3:], np.float64)
    pos = 0

    def take(nb):
        nonlocal pos
        chunk = data[pos:pos + nb]
        pos += nb
        return chunk

    out = dict(count=n, active_count=active, sh_degree=degree, profile_id=profile)
    if profile == 1:
        out["means"] = np.frombuffer(take(12 * n), "<f4").reshape(n, 3).copy()
        out["log_scales"] = np.frombuffer(take(12 * n), "<f4").reshape(n, 3).copy()
        out["quaternions"] = np.frombuffer(take(16 * n), "<f4").reshape(n, 4).copy()
        out["logit_opacities"] = np.frombuffer(take(4 * n), "<f4").copy()
        out["sh_coeffs"] = np.frombuffer(take(12 * B * n), "<f4").reshape(n, 3, B).copy()
        out["light_visibility"] = np.frombuffer(take(4 * n), "<f4").copy()
        out["object_ids"] = np.frombuffer(take(4 * n), "<i4").copy()
        return out
    c = np.frombuffer(take(6 * n), "<u2").reshape(n, 3)
    out["means"] = dequantize(c, lo, hi, 16).astype(np.float32)
    b, qlo, qhi = QUANT[LOG_SCALES]
    out["log_scales"] = dequantize(np.frombuffer(take(3 * n), "<u1").reshape(n, 3), qlo, qhi, b).astype(np.float32)
    b, qlo, qhi = QUANT[QUATERNIONS]
    q = unpack_lsb(take((4 * n * b + 7) // 8), b, 4 * n).reshape(n, 4)
    out["quaternions"] = dequantize(q, qlo, qhi, b).astype(np.float32)
    b, qlo, qhi = QUANT[LOGIT_OPACITIES]
    out["logit_opacities"] = dequantize(np.frombuffer(take(n), "<u1"), qlo, qhi, b).astype(np.float32)
    sh = np.zeros((n, 3, B), np.float32)
    b, qlo, qhi = QUANT[SH_DC]
    sh[:, :, 0] = dequantize(np.frombuffer(take(3 * n), "<u1").reshape(n, 3), qlo, qhi, b)
    if B > 1:
        b, qlo, qhi = QUANT[SH_REST]
        sh[:, :, 1:] = dequantize(np.frombuffer(take(3 * (B - 1) * n), "<u1").reshape(n, 3, B - 1), qlo, qhi, b)
    out["sh_coeffs"] = sh
    out["light_visibility"] = unpack_lsb(take((n + 7) // 8), 1, n).astype(np.float32)
    ids, _ = leb128_decode(data, n, pos)
    out["object_ids"] = ids.astype(np.int32)
    return out


def light_visibility_payload(vis) -> bytes:
    """ref protocol/packets.py:73-76."""
    v = np.asarray(vis)
    return struct.pack("<I", v.size) + pack_lsb((v >= 0.5).astype(np.uint32), 1)
