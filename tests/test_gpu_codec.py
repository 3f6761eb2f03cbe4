"""GPU encoders vs the reference's bytes (golden vectors) -- bit-exact."""

import numpy as np
import pytest

from conftest import case_model, load_cases
from gpu_util import require_gpu

pytestmark = pytest.mark.gpu

DELTAS = [c for c in load_cases("codec_cases") if c["kind"] == "delta"]
SNAPS = [c for c in load_cases("codec_cases") if c["kind"] == "snapshot"]


@pytest.mark.parametrize("c", DELTAS, ids=[c["name"] for c in DELTAS])
def test_gpu_delta_bit_exact(c):
    require_gpu()
    from paper_2604_02851_b200.protocol import encode_delta
    base = c.a("base") if c.has("base") else None
    for comp in (0, 1):
        got, nb = encode_delta(c["attr"], c.a("cur"), base, c["gate"], comp)
        assert got == c.a(f"payload{comp}").tobytes(), comp
        if base is not None:
            assert nb.dtype == np.float32
            np.testing.assert_array_equal(nb, c.a("new_base"))


@pytest.mark.parametrize("c", SNAPS, ids=[c["name"] for c in SNAPS])
def test_gpu_snapshot_bit_exact(c):
    require_gpu()
    from paper_2604_02851_b200.model import GaussianModel
    from paper_2604_02851_b200.protocol import QuantizationProfile, encode_snapshot
    m = case_model(c)
    model = GaussianModel(m.means, m.log_scales, m.quaternions, m.logit_opacities, m.sh_coeffs,
                          m.light_visibility, m.object_ids, m.active_count, m.sh_degree)
    for prof in (0, 1):
        for comp in (0, 1):
            got, (bm, bl) = encode_snapshot(model, QuantizationProfile(prof, comp), return_baselines=True)
            assert got == c.a(f"payload_p{prof}c{comp}").tobytes(), (prof, comp)
            if prof == 0 and c.has("dec_means"):
                np.testing.assert_array_equal(bm, c.a("dec_means"))
                np.testing.assert_array_equal(bl, c.a("dec_log_scales"))
            if prof == 1:
                np.testing.assert_array_equal(bm, m.means)


def test_gpu_delta_dual_ledger_random_walk():
    """ref pkg/tests/test_protocol.py:360-392 restated: the GPU encoder's
    baseline equals the oracle's bit for bit over 50 ticks."""
    require_gpu()
    from oracle import codec as oc
    from paper_2604_02851_b200.protocol import encode_delta
    rng = np.random.default_rng(15)
    n = 600
    cur = rng.uniform(-3, 3, (n, 3)).astype(np.float32)
    base_gpu = cur.copy()
    base_ref = cur.copy()
    for tick in range(50):
        moved = rng.random(n) < (0.3 if tick % 7 else 0.9)
        cur[moved] += rng.normal(0, 0.01, (int(moved.sum()), 3)).astype(np.float32)
        p_gpu, base_gpu = encode_delta(0, cur, base_gpu, 1e-3, 0)
        p_ref, base_ref = oc.delta_payload(0, cur, base_ref, 1e-3, 0)
        assert p_gpu == p_ref
        np.testing.assert_array_equal(base_gpu, base_ref)


def test_gpu_large_delta_and_snapshot_match_oracle():
    """Sizes beyond the fixtures: 300k rows, both residual modes, all attributes."""
    require_gpu()
    from oracle import codec as oc
    from paper_2604_02851_b200.model import GaussianModel
    from paper_2604_02851_b200.protocol import QuantizationProfile, encode_delta, encode_snapshot
    rng = np.random.default_rng(5)
    n = 300_000
    base = rng.uniform(-4, 4, (n, 3)).astype(np.float32)
    for frac in (0.2, 0.9):
        cur = base.copy()
        mv = rng.random(n) < frac
        cur[mv] += rng.normal(0, 0.02, (int(mv.sum()), 3)).astype(np.float32)
        for attr in (0, 1):
            g, gb = encode_delta(attr, cur, base, None, 0)
            r, rb = oc.delta_payload(attr, cur, base, None, 0)
            assert g == r
            np.testing.assert_array_equal(gb, rb)
    sh = rng.uniform(-1.2, 1.2, (n, 3, 16)).astype(np.float32)
    for attr, x in ((2, rng.normal(0, 0.5, (n, 4)).astype(np.float32)), (3, rng.uniform(-9, 9, n).astype(np.float32)),
                    (4, sh[:, :, 0]), (5, sh[:, :, 1:]), (6, rng.random(n).astype(np.float32))):
        assert encode_delta(attr, x, None, None, 0)[0] == oc.delta_payload(attr, x, None, None, 0)[0]
    q = rng.normal(size=(n, 4))
    model = GaussianModel(base, rng.uniform(-6, 1, (n, 3)).astype(np.float32),
                          (q / np.linalg.norm(q, axis=1, keepdims=True)).astype(np.float32),
                          rng.uniform(-6, 6, n).astype(np.float32), sh, (rng.random(n) > 0.5).astype(np.float32),
                          rng.integers(0, 300, n).astype(np.int32), n - 1000, 3)
    for prof in (0, 1):
        g = encode_snapshot(model, QuantizationProfile(prof, 0))
        r = oc.snapshot_payload(model.means, model.log_scales, model.quaternions, model.logit_opacities,
                                model.sh_coeffs, model.light_visibility, model.object_ids, model.active_count, 3,
                                prof, 0)
        assert g == r


def test_gpu_light_visibility_packet():
    require_gpu()
    from oracle import codec as oc
    from paper_2604_02851_b200.protocol import encode_light_visibility
    rng = np.random.default_rng(2)
    for n in (0, 1, 10, 33, 1000, 12345):
        v = rng.random(n).astype(np.float32)
        assert encode_light_visibility(v) == oc.light_visibility_payload(v)


@pytest.mark.parametrize("degree", [0, 1, 3])
def test_gpu_batched_delta_tick_matches_oracle(degree):
    """DeltaTicker (one library call per tick, SH DC/rest read strided in
    place, residual baselines advanced in HBM) == the oracle's per-attribute
    payloads and baselines over a short walk with changing sparsity."""
    require_gpu()
    import torch
    from oracle import codec as oc
    from paper_2604_02851_b200 import synth
    from paper_2604_02851_b200.model import DeviceModel
    from paper_2604_02851_b200.protocol import DeltaTicker, PayloadBuffer
    rng = np.random.default_rng(9 + degree)
    n = 70_001
    host = synth.random_field(n, degree, 320, 180, seed=3)
    dm = DeviceModel.from_host(host, 0)
    a = dm.active_count
    base = {0: host.means[:a].copy(), 1: host.log_scales[:a].copy()}
    dbase = {k: torch.from_numpy(v).cuda() for k, v in base.items()}
    attrs = [0, 1, 2, 3, 4] + ([5] if degree else [])
    ticker = DeltaTicker(dm, dbase, {k: PayloadBuffer(64, dm.device) for k in attrs})
    for tick, frac in enumerate((0.0, 0.05, 0.6, 1.0)):
        for t in (dm.means, dm.log_scales, dm.sh_coeffs):
            mv = torch.from_numpy(rng.random(n) < frac).cuda()
            t[mv] += torch.randn_like(t[mv]) * 0.01
        for sub in (attrs, attrs[::2]):
            ticker(sub)
            got = ticker.read(sub)
            h = dm.to_host()
            for attr, g in zip(sub, got):
                if attr in (0, 1):
                    cur = h.means if attr == 0 else h.log_scales
                    r, base[attr] = oc.delta_payload(attr, cur[:a], base[attr], None, 0)
                    np.testing.assert_array_equal(dbase[attr].cpu().numpy(), base[attr])
                else:
                    x = {2: h.quaternions, 3: h.logit_opacities, 4: h.sh_coeffs[:, :, 0],
                         5: h.sh_coeffs[:, :, 1:]}[attr][:a]
                    r = oc.delta_payload(attr, x, None, None, 0)[0]
                assert g == r, (tick, attr)


def test_gpu_delta_gate_boundary_exact():
    """Residuals within a few float32 ulps of the gating threshold (the
    float32 fast path defers to the exact float64 test there), gates equal to
    a residual, zero and negative gates, both modes."""
    require_gpu()
    from oracle import codec as oc
    from paper_2604_02851_b200.protocol import encode_delta
    rng = np.random.default_rng(17)
    n = 5000
    for gate in (1e-3, float(np.float32(1e-3)), 2.5e-4, 0.0, -1.0):
        g32 = np.float32(gate) if gate > 0 else np.float32(1e-3)
        near = np.array([g32, np.nextafter(g32, np.float32(0)), np.nextafter(g32, np.float32(1)),
                         np.nextafter(np.nextafter(g32, np.float32(0)), np.float32(0))], np.float32)
        for frac in (0.1, 0.8):
            base = rng.uniform(-2, 2, (n, 3)).astype(np.float32)
            cur = base.copy()
            mv = rng.random(n) < frac
            cur[mv] += rng.normal(0, 0.01, (int(mv.sum()), 3)).astype(np.float32)
            # rows whose largest |residual| sits on the gate (base 0 keeps the residual exact)
            idx = rng.choice(n, 400, replace=False)
            base[idx] = 0.0
            cur[idx] = rng.choice(near, (400, 3)) * rng.choice([-1, 1], (400, 3)).astype(np.float32)
            for attr in (0, 1):
                g, gb = encode_delta(attr, cur, base, gate, 0)
                r, rb = oc.delta_payload(attr, cur, base, gate, 0)
                assert g == r, (gate, frac, attr)
                np.testing.assert_array_equal(gb, rb)


def test_gpu_delta_emitter_server_ticks_match_oracle():
    """DeltaEmitter over 31 server ticks (zlib payloads) of a model that moves
    like an optimised one, vs the oracle's encode_delta + baseline advance
    for the same schedule; a replica fed the payloads tracks the baselines."""
    require_gpu()
    import torch
    from oracle import codec as oc
    from paper_2604_02851_b200 import synth
    from paper_2604_02851_b200.model import DeviceModel
    from paper_2604_02851_b200.protocol import DeltaEmitter, DeviceBaselines, apply_delta, due_attributes
    rng = np.random.default_rng(12)
    host = synth.random_field(20_000, 2, 320, 180, seed=4)
    host.active_count = 19_000
    a = host.active_count
    dm = DeviceModel.from_host(host, 0)
    base = DeviceBaselines()
    base.reset_from_model(dm, 1)
    em = DeltaEmitter(dm, base)
    replica = dm.clone()
    rbase = DeviceBaselines()
    rbase.reset_from_model(replica, 1)
    hb_m, hb_l = host.means.copy(), host.log_scales.copy()
    for tick in range(31):
        with torch.no_grad():
            for t, s in ((dm.means, 2e-3), (dm.log_scales, 3e-3), (dm.quaternions, 1e-2), (dm.sh_coeffs, 1e-2)):
                mv = torch.from_numpy(rng.random(t.shape[0]) < 0.4).cuda()
                t[:a][mv[:a]] += torch.randn_like(t[:a][mv[:a]]) * s
        out = em.tick(tick)
        assert [p[0] for p in out] == [int(x) for x in due_attributes(tick, sh_degree=2)]
        h = dm.to_host()
        for attr, payload in out:
            if attr == 0:
                ref, hb_m[:a] = oc.delta_payload(0, h.means[:a], hb_m[:a], None, 1)
            elif attr == 1:
                ref, hb_l[:a] = oc.delta_payload(1, h.log_scales[:a], hb_l[:a], None, 1)
            else:
                x = {2: h.quaternions, 3: h.logit_opacities, 4: h.sh_coeffs[:, :, 0], 5: h.sh_coeffs[:, :, 1:]}[attr]
                ref = oc.delta_payload(attr, x[:a], None, None, 1)[0]
            assert payload == ref, (tick, attr)
            assert apply_delta(replica, rbase, payload, 1, 1)
        np.testing.assert_array_equal(base.means.cpu().numpy(), hb_m)
        np.testing.assert_array_equal(base.log_scales.cpu().numpy(), hb_l)
        np.testing.assert_array_equal(rbase.means.cpu().numpy(), hb_m)
        np.testing.assert_array_equal(replica.means[:a].cpu().numpy(), hb_m[:a])


def test_gpu_ticker_read_async_matches_read():
    """read_async (bound-sized copies, no host sync) returns the same bytes as read()."""
    require_gpu()
    import torch
    from paper_2604_02851_b200 import synth
    from paper_2604_02851_b200.model import DeviceModel
    from paper_2604_02851_b200.protocol import DeltaTicker, PayloadBuffer
    host = synth.random_field(30_000, 1, 320, 180, seed=8)
    dm = DeviceModel.from_host(host, 0)
    base = {0: (dm.means - 1e-3).contiguous(), 1: dm.log_scales.clone()}
    t = DeltaTicker(dm, base, {k: PayloadBuffer(64, dm.device) for k in range(7)})
    attrs = [0, 1, 3, 4, 5]
    t(attrs)
    p1 = t.read_async(attrs)
    sync = t.read(attrs)
    t(attrs)  # second tick while the first readback may be pending
    p2 = t.read_async(attrs)
    assert p1.result() == sync
    assert p2.result() == t.read(attrs)


@pytest.mark.parametrize("ids", ["one_byte", "multi_byte", "negative", "one_long"])
def test_gpu_snapshot_object_id_varints(ids):
    """The snapshot's object-id section: one-byte varints are written in
    place, any longer id switches the batch to the scanned offsets (a
    device-side flag) -- every case byte-exact vs the oracle."""
    require_gpu()
    from oracle import codec as oc
    from paper_2604_02851_b200 import synth
    from paper_2604_02851_b200.protocol import QuantizationProfile, encode_snapshot
    n = 70_001
    m = synth.random_field(n, 2, 320, 192, seed=3)
    rng = np.random.default_rng(4)
    if ids == "one_byte":
        m.object_ids = rng.integers(0, 128, n).astype(np.int32)
    elif ids == "multi_byte":
        m.object_ids = rng.integers(0, 1 << 20, n).astype(np.int32)
    elif ids == "negative":
        m.object_ids = rng.integers(-3, 3, n).astype(np.int32)
    else:
        m.object_ids = np.zeros(n, np.int32)
        m.object_ids[n - 5] = 300  # one two-byte id at the very end
    got = encode_snapshot(m, QuantizationProfile(0, 0))
    ref = oc.snapshot_payload(m.means, m.log_scales, m.quaternions, m.logit_opacities, m.sh_coeffs,
                              m.light_visibility, m.object_ids, m.active_count, m.sh_degree, 0, 0)
    assert got == ref
