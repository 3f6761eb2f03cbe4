"""Client ingestion: decode_delta / apply_delta /
decode_snapshot on a device replica vs the reference.

The expectations are the unmodified reference's own results
(tests/golden/make_golden.py::ingest_cases): the replica and baselines after
apply_delta, decode_snapshot's arrays, and the (exception type, message) for
corrupted payloads.  Bit-exact throughout.  The host-side header parser is
checked on CPU; everything else runs through the C ABI on the GPU.
"""

import struct

import numpy as np
import pytest

from conftest import load_cases
from gpu_util import require_gpu

CASES = load_cases("ingest_cases")
GROUPS = {c["group"]: c for c in CASES if c["kind"] == "replica"}
DELTAS = [c for c in CASES if c["kind"] == "delta"]
SNAPS = [c for c in CASES if c["kind"] == "snapshot"]
SNAP_ERRORS = [c for c in CASES if c["kind"] == "snapshot_error"]
FIELDS = ("means", "log_scales", "quaternions", "logit_opacities", "sh_coeffs", "light_visibility", "object_ids")
# checked on the device (need the block's bytes) or against the replica
DEVICE_CHECKED = {"sparse delta index out of range", "delta codes truncated", "delta covers 39 rows, active is 40",
                  "varint too long", "truncated varint"}


def _exc_name(e):
    return type(e).__name__


@pytest.mark.parametrize("c", [c for c in DELTAS if "error" in c], ids=lambda c: c["name"])
def test_host_parser_errors_match_reference(c):
    """Everything decidable from sizes raises on the host exactly like the
    reference (type and message); the rest must reach the device checks."""
    from paper_2604_02851_b200.protocol.ingest import parse_delta
    try:
        parse_delta(c.a("payload").tobytes())
    except Exception as e:  # noqa: BLE001
        assert (_exc_name(e), str(e)) == (c["error"], c["message"])
        return
    assert c["message"] in DEVICE_CHECKED, c["name"]


def _replica(g):
    import torch
    from paper_2604_02851_b200.model import DeviceModel
    from paper_2604_02851_b200.protocol import DeviceBaselines
    dev = torch.device("cuda", 0)
    t = lambda k: torch.from_numpy(np.array(g.a(k))).to(dev)
    m = DeviceModel(*(t(k) for k in FIELDS), g["active"], g["degree"])
    b = DeviceBaselines(t("base_means"), t("base_log_scales"), 3)
    return m, b


@pytest.mark.gpu
@pytest.mark.parametrize("c", DELTAS, ids=lambda c: c["name"])
def test_gpu_apply_delta_matches_reference(c):
    require_gpu()
    from paper_2604_02851_b200.protocol import apply_delta
    g = GROUPS[c["group"]]
    m, b = _replica(g)
    payload = c.a("payload").tobytes()
    if "error" in c:
        with pytest.raises(Exception) as ei:
            apply_delta(m, b, payload, 3, 3)
        assert (_exc_name(ei.value), str(ei.value)) == (c["error"], c["message"])
        for k in FIELDS:  # nothing written
            np.testing.assert_array_equal(getattr(m, k).cpu().numpy(), g.a(k), err_msg=k)
        np.testing.assert_array_equal(b.means.cpu().numpy(), g.a("base_means"))
        return
    assert apply_delta(m, b, payload, 3, 3) is True
    f = c["field"]
    np.testing.assert_array_equal(getattr(m, f).cpu().numpy(), c.a(f"after_{f}"))
    np.testing.assert_array_equal(b.means.cpu().numpy(), c.a("after_base_means"))
    np.testing.assert_array_equal(b.log_scales.cpu().numpy(), c.a("after_base_log_scales"))
    for k in FIELDS:
        if k != f:
            np.testing.assert_array_equal(getattr(m, k).cpu().numpy(), g.a(k), err_msg=k)


@pytest.mark.gpu
def test_gpu_apply_delta_stale_epoch_untouched():
    require_gpu()
    from paper_2604_02851_b200.protocol import apply_delta
    c = [c for c in DELTAS if c["name"].startswith("means_sparse_300")][0]
    m, b = _replica(GROUPS[c["group"]])
    assert apply_delta(m, b, c.a("payload").tobytes(), 2, 3) is False
    np.testing.assert_array_equal(m.means.cpu().numpy(), GROUPS[c["group"]].a("means"))


@pytest.mark.gpu
@pytest.mark.parametrize("c", [c for c in DELTAS if "error" not in c][:40], ids=lambda c: c["name"])
def test_gpu_decode_delta_matches_oracle(c):
    """decode_delta's DeltaUpdate (indices, float64 values) vs the oracle,
    itself pinned to the reference's payloads (test_oracle_golden)."""
    require_gpu()
    from oracle import codec as oc
    from paper_2604_02851_b200.protocol import decode_delta
    payload = c.a("payload").tobytes()
    got = decode_delta(payload)
    ref = oc.delta_unpack(payload)
    assert (got.attribute_id, got.mode, got.count, got.dims) == (ref["attr"], ref["mode"], ref["count"], ref["dims"])
    if ref["indices"] is None:
        assert got.indices is None
    else:
        np.testing.assert_array_equal(got.indices, ref["indices"])
    np.testing.assert_array_equal(got.values.reshape(ref["values"].shape), ref["values"])


def _put_block(payload: bytes, head: int, block: bytes) -> bytes:
    return payload[:head] + struct.pack("<I", len(block)) + block


@pytest.mark.gpu
def test_gpu_varint_edge_cases():
    """Blocks that pass the size bound but break decode_varints
    (quantize.py:74-96): 11-byte varints ("too long" at the 10th byte),
    a run that ends before k varints ("truncated"), a 10-continuation tail
    ("too long"), and gaps of 1-3 bytes decoding to the right indices."""
    require_gpu()
    from paper_2604_02851_b200.protocol import apply_delta
    c = [c for c in DELTAS if c["name"].startswith("means_sparse_300_c0")][0]
    g = GROUPS[c["group"]]
    payload = c.a("payload").tobytes()
    assert payload[1] == 1
    k = struct.unpack_from("<I", payload, 16)[0]
    assert k >= 4
    cases = [
        (b"\x81" * 10 + b"\x01" + bytes(6 * k + 8), ValueError, "varint too long"),  # first varint 11 bytes
        (b"\x00\x00" + b"\x80" * 10 + bytes(6 * k), ValueError, "varint too long"),   # third varint too long
        (b"\x00" * (k - 1) + b"\x80\x80", ValueError, "truncated varint"),          # k-th varint runs off the end
        (b"\x00" * (k - 1) + b"\x80" * 10, ValueError, "varint too long"),          # ... after 10 continuation bytes
    ]
    for block, exc, msg in cases:
        m, b = _replica(g)
        with pytest.raises(exc, match=msg):
            apply_delta(m, b, _put_block(payload, 20, block), 3, 3)
        np.testing.assert_array_equal(m.means.cpu().numpy(), g.a("means"))


@pytest.mark.gpu
def test_gpu_large_roundtrip_encode_apply():
    """300k-row replica: GPU-encoded deltas of every attribute applied on the
    GPU equal the oracle's apply (both peers bit-identical), dense and sparse."""
    require_gpu()
    import torch
    from oracle import codec as oc
    from paper_2604_02851_b200 import synth
    from paper_2604_02851_b200.model import DeviceModel
    from paper_2604_02851_b200.protocol import DeviceBaselines, apply_delta, encode_delta
    rng = np.random.default_rng(3)
    n = 300_000
    host = synth.random_field(n, 3, 640, 360, seed=2)
    host.active_count = n - 5000
    a = host.active_count
    dm = DeviceModel.from_host(host, 0)
    base = DeviceBaselines()
    base.reset_from_model(dm, 1)
    hb_means = host.means.copy()
    for frac in (0.05, 0.9):
        cur = hb_means[:a].copy()
        mv = rng.random(a) < frac
        cur[mv] += rng.normal(0, 0.01, (int(mv.sum()), 3)).astype(np.float32)
        payload, _ = encode_delta(0, cur, hb_means[:a], None, 1)
        assert apply_delta(dm, base, payload, 1, 1)
        upd = oc.delta_unpack(payload)
        oc.apply_residual(hb_means[:a], upd["indices"], upd["values"])
        np.testing.assert_array_equal(base.means.cpu().numpy(), hb_means)
        np.testing.assert_array_equal(dm.means[:a].cpu().numpy(), hb_means[:a])
    B = 16
    vals = {2: rng.normal(0, 0.5, (a, 4)).astype(np.float32), 3: rng.uniform(-9, 9, a).astype(np.float32),
            4: rng.uniform(-4, 4, (a, 3)).astype(np.float32), 5: rng.uniform(-1, 1, (a, 3, B - 1)).astype(np.float32),
            6: (rng.random(a) > 0.5).astype(np.float32)}
    for attr, v in vals.items():
        payload, _ = encode_delta(attr, v, None, None, 0)
        assert apply_delta(dm, base, payload, 1, 1)
        ref = oc.delta_unpack(payload)["values"].astype(np.float32)
        got = {2: dm.quaternions, 3: dm.logit_opacities, 4: dm.sh_coeffs[:, :, 0], 5: dm.sh_coeffs[:, :, 1:],
               6: dm.light_visibility}[attr][:a].cpu().numpy()
        np.testing.assert_array_equal(got.reshape(a, -1), ref.reshape(a, -1))
    torch.cuda.synchronize()


@pytest.mark.gpu
@pytest.mark.parametrize("c", SNAPS, ids=lambda c: c["name"])
def test_gpu_decode_snapshot_matches_reference(c):
    require_gpu()
    from paper_2604_02851_b200.protocol import decode_snapshot
    m, info = decode_snapshot(c.a("payload").tobytes())
    assert (m.active_count, m.sh_degree) == (c["active"], c["degree"])
    for k in FIELDS:
        np.testing.assert_array_equal(getattr(m, k).cpu().numpy(), c.a(f"dec_{k}"), err_msg=k)
    np.testing.assert_array_equal(info["aabb_lo"], c.a("aabb_lo"))
    np.testing.assert_array_equal(info["aabb_hi"], c.a("aabb_hi"))


@pytest.mark.gpu
@pytest.mark.parametrize("c", SNAP_ERRORS, ids=lambda c: c["name"])
def test_gpu_decode_snapshot_errors_match_reference(c):
    require_gpu()
    from paper_2604_02851_b200.protocol import decode_snapshot
    with pytest.raises(Exception) as ei:
        decode_snapshot(c.a("payload").tobytes())
    assert (_exc_name(ei.value), str(ei.value)) == (c["error"], c["message"])


def test_due_attributes_follow_server_schedule():
    """ref server.py:57-74, 89-91, 488-493, 352-354."""
    from paper_2604_02851_b200.protocol import due_attributes
    assert [int(a) for a in due_attributes(0)] == [0, 1, 2, 3, 4, 5]
    assert [int(a) for a in due_attributes(1)] == [0, 1, 3, 4]
    assert [int(a) for a in due_attributes(10)] == [0, 1, 2, 3, 4]
    assert [int(a) for a in due_attributes(30)] == [0, 1, 2, 3, 4, 5]
    assert [int(a) for a in due_attributes(7, appended=True)] == [0, 1, 2, 3, 4, 5]
    assert [int(a) for a in due_attributes(0, sh_degree=0)] == [0, 1, 2, 3, 4]
