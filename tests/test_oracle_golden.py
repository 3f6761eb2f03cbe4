"""Pin the CPU oracle against vectors produced by the unmodified reference.

CPU-only (no GPU).  Bit-exact for every encoder byte and baseline; float64
tolerances for the renderer / backward / optimizer restatements.
"""

import json
import struct

import numpy as np
import pytest

from conftest import GOLDEN, NS, case_model, load_cases
from oracle import adam as oadam
from oracle import codec as oc
from oracle import dynamics as odyn
from oracle import raster as orr

WIRE = GOLDEN / "wire"
MANIFEST = json.loads((WIRE / "manifest.json").read_text())


def frame_payload(name):
    buf = (WIRE / f"{name}.bin").read_bytes()
    assert buf[:2] == b"GS"
    ptype, epoch, n = struct.unpack_from("<BII", buf, 2)
    return buf[11:11 + n]


# ---------------------------------------------------------------- wire fixtures
def _fixture_model_arrays():
    """Same draws as ref pkg/scripts/make_golden_packets.py:48-61."""
    rng = np.random.default_rng(2024)
    n, B = 8, 4
    means = rng.uniform(-2, 2, (n, 3)).astype(np.float32)
    ls = rng.uniform(-3, -1, (n, 3)).astype(np.float32)
    q = rng.normal(size=(n, 4))
    q = (q / np.linalg.norm(q, axis=-1, keepdims=True)).astype(np.float32)
    logits = rng.uniform(-1, 2, n).astype(np.float32)
    sh = rng.uniform(-0.4, 0.4, (n, 3, B)).astype(np.float32)
    vis = (rng.random(n) > 0.3).astype(np.float32)
    ids = np.array([0, 0, 1, 1, 1, 2, 2, 2], np.int32)
    return means, ls, q, logits, sh, vis, ids


@pytest.mark.parametrize("name,profile", [("snapshot_quantized", 0), ("snapshot_lossless", 1)])
def test_wire_snapshot_fixture_bytes(name, profile):
    means, ls, q, logits, sh, vis, ids = _fixture_model_arrays()
    src = MANIFEST[name]["source_model"]
    np.testing.assert_array_equal(means.astype(np.float64), src["means"])
    got = oc.snapshot_payload(means, ls, q, logits, sh, vis, ids, 6, 1, profile, 1)
    assert got == frame_payload(name)


def test_wire_delta_fixture_bytes():
    """Re-encode the delta trio from the draws of make_golden_packets.py:153-185."""
    rng = np.random.default_rng(77)
    base = rng.uniform(-1, 1, (6, 3)).astype(np.float32)
    cur = base.copy()
    cur[1] += np.float32([0.05, 0.0, -0.02])
    cur[4, 2] += np.float32(0.004)
    got, nb = oc.delta_payload(oc.MEANS, cur, base, 1e-3)
    assert got == frame_payload("delta_sparse_residual")
    np.testing.assert_array_equal(nb.astype(np.float64), MANIFEST["delta_sparse_residual"]["expected_baseline_after"])
    dense = (base + rng.uniform(0.01, 0.03, base.shape)).astype(np.float32)
    got, nb = oc.delta_payload(oc.MEANS, dense, base, 1e-3)
    assert got == frame_payload("delta_dense_residual")
    np.testing.assert_array_equal(nb.astype(np.float64), MANIFEST["delta_dense_residual"]["expected_baseline_after"])
    ops = rng.uniform(-2, 3, 6).astype(np.float32)
    got, _ = oc.delta_payload(oc.LOGIT_OPACITIES, ops)
    assert got == frame_payload("delta_absolute")
    upd = oc.delta_unpack(got)
    np.testing.assert_array_equal(upd["values"].reshape(6), MANIFEST["delta_absolute"]["expected_values"])


def test_wire_light_visibility_fixture():
    vis = np.array(MANIFEST["light_visibility"]["visibility"], np.float32)
    assert oc.light_visibility_payload(vis) == frame_payload("light_visibility")


def test_varints_match_reference_examples():
    vals = np.array([0, 1, 127, 128, 300, 2 ** 21, 2 ** 35], np.uint64)
    enc = oc.leb128(vals)
    dec, off = oc.leb128_decode(enc, len(vals))
    assert off == len(enc)
    np.testing.assert_array_equal(dec, vals)
    assert oc.leb128([300]) == b"\xac\x02"


# ---------------------------------------------------------------- codec vectors
DELTAS = [c for c in load_cases("codec_cases") if c["kind"] == "delta"]
SNAPS = [c for c in load_cases("codec_cases") if c["kind"] == "snapshot"]


@pytest.mark.parametrize("c", DELTAS, ids=[c["name"] for c in DELTAS])
def test_oracle_delta_bit_exact(c):
    base = c.a("base") if c.has("base") else None
    for comp in (0, 1):
        got, nb = oc.delta_payload(c["attr"], c.a("cur"), base, c["gate"], comp)
        assert got == c.a(f"payload{comp}").tobytes()
        if base is not None:
            assert nb.dtype == np.float32
            np.testing.assert_array_equal(nb, c.a("new_base"))


@pytest.mark.parametrize("c", SNAPS, ids=[c["name"] for c in SNAPS])
def test_oracle_snapshot_bit_exact(c):
    m = case_model(c)
    for prof in (0, 1):
        for comp in (0, 1):
            got = oc.snapshot_payload(m.means, m.log_scales, m.quaternions, m.logit_opacities, m.sh_coeffs,
                                      m.light_visibility, m.object_ids, m.active_count, m.sh_degree, prof, comp)
            assert got == c.a(f"payload_p{prof}c{comp}").tobytes(), (prof, comp)
    if c.has("dec_means"):
        dec = oc.snapshot_dequant(c.a("payload_p0c1").tobytes())
        np.testing.assert_array_equal(dec["means"], c.a("dec_means"))
        np.testing.assert_array_equal(dec["log_scales"], c.a("dec_log_scales"))


# ---------------------------------------------------------------- raster vectors
RASTER = load_cases("raster_cases")


def case_camera(c):
    pose = c.a("pose")
    intr = NS(width=c["W"], height=c["H"], fov_y=c["fov"], near=c["near"])
    return orr.camera(NS(position=pose[:3], quaternion=pose[3:]), intr)


def case_light(c):
    return dict(direction=c.a("light_dir"), intensity=c.a("light_int"),
                ambient=c.a("ambient") if c.has("ambient") else None)


@pytest.mark.parametrize("c", RASTER, ids=[c["name"] for c in RASTER])
def test_oracle_prepare_matches_reference(c):
    m = case_model(c)
    cam = case_camera(c)
    sub = c.a("subset") if c.has("subset") else None
    p = orr.prepare(m, cam, case_light(c), sub, c["cutoff"])
    np.testing.assert_array_equal(p["rows"], c.a("rows"))
    np.testing.assert_array_equal(p["order"], c.a("order"))
    np.testing.assert_array_equal(p["rect"], c.a("windows"))  # measured agreement: 100%
    np.testing.assert_allclose(p["depth"], c.a("depth"), rtol=1e-15, atol=0)
    np.testing.assert_allclose(p["mu2d"], c.a("mu2d"), rtol=1e-13, atol=1e-12)
    for k in ("Sigma2d", "Sigma3d"):  # the reference's [0,1]/[1,0] entries differ by rounding
        ref = c.a(k)
        np.testing.assert_allclose(p[k], ref, rtol=1e-12, atol=1e-13 * np.abs(ref).max(initial=1.0))
    np.testing.assert_allclose(p["radius"], c.a("radius"), rtol=1e-13)
    np.testing.assert_allclose(p["color_pre"], c.a("color_pre"), rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(p["s"], c.a("s"), rtol=1e-12, atol=1e-13)


@pytest.mark.parametrize("c", RASTER, ids=[c["name"] for c in RASTER])
def test_oracle_render_and_backward_match_reference(c):
    m = case_model(c)
    cam = case_camera(c)
    sub = c.a("subset") if c.has("subset") else None
    L, g, img = orr.backward(m, cam, case_light(c), c.a("gt"), c.a("bg"), sub, c["cutoff"])
    np.testing.assert_allclose(img, c.a("image"), rtol=0, atol=1e-12)
    assert abs(L - c["loss"]) <= 1e-12
    _, T = orr.render(m, cam, case_light(c), c.a("bg"), sub, c["cutoff"])
    np.testing.assert_allclose(T, c.a("T"), rtol=0, atol=1e-12)
    for name in ("means", "log_scales", "quaternions", "logit_opacities", "sh_coeffs"):
        ref = c.a(f"g_{name}")
        scale = max(np.abs(ref).max(initial=0.0), 1e-30)
        assert np.abs(g[name] - ref).max(initial=0.0) <= 1e-9 * scale, name


def test_oracle_tile_bins_consistent_with_windows():
    c = [c for c in RASTER if c["name"] == "medium"][0]
    m = case_model(c)
    cam = case_camera(c)
    p = orr.prepare(m, cam, case_light(c), None, True)
    b = orr.tile_bins(p, c["W"], c["H"])
    tw = -(-c["W"] // 16)
    rect = p["rect"][p["order"]]
    for t in range(b["ranges"].shape[0]):
        lo, hi = b["ranges"][t]
        ranks = b["pair_rank"][lo:hi]
        assert np.all(np.diff(ranks) > 0)
        tx, ty = t % tw, t // tw
        X0, Y0 = tx * 16, ty * 16
        hit = (rect[:, 0] < X0 + 16) & (rect[:, 1] > X0) & (rect[:, 2] < Y0 + 16) & (rect[:, 3] > Y0) & \
              (rect[:, 0] < rect[:, 1]) & (rect[:, 2] < rect[:, 3])
        np.testing.assert_array_equal(ranks, np.flatnonzero(hit))


def test_det_exp_accuracy():
    x = np.linspace(-30, 12, 200001)
    rel = np.abs(orr.det_exp(x) - np.exp(x)) / np.exp(x)
    assert rel.max() < 4e-16


# ---------------------------------------------------------------- optimizer step
STEPS = load_cases("step_cases")


@pytest.mark.parametrize("c", STEPS, ids=[f"deg{c['degree']}" for c in STEPS])
def test_oracle_step_trajectory(c):
    m = case_model(c, "init_")
    B = m.sh_coeffs.shape[2]
    st = oadam.AdamState(m.active_count, B, scene_extent=c["scene_extent"])
    light = dict(direction=c.a("light_dir"), intensity=c.a("light_int"), ambient=c.a("ambient"))
    intr = NS(width=c["W"], height=c["H"], fov_y=c["fov"], near=c["near"])
    cams = [orr.camera(NS(position=p[:3], quaternion=p[3:]), intr) for p in c.a("poses")]
    for it in range(c["steps"]):
        total, lsum = None, 0.0
        for cam, gt in zip(cams, c.a("gts")):
            L, g, _ = orr.backward(m, cam, light, gt, c.a("bg"))
            lsum += L
            total = g if total is None else {k: total[k] + g[k] for k in g}
        oadam.apply(m, st, total, len(cams))
        assert abs(lsum / len(cams) - c.a("losses")[it]) < 1e-9
        for k in oadam.GROUPS:
            np.testing.assert_allclose(getattr(m, k), c.a(f"after{it}_{k}"), rtol=0, atol=2e-6, err_msg=k)
    np.testing.assert_array_equal(st.age, c.a("age"))
    np.testing.assert_allclose(st.grad_ema, c.a("grad_ema"), rtol=1e-6)


# ---------------------------------------------------------------- dynamics
DYN = load_cases("dyn_cases")


@pytest.mark.parametrize("c", DYN, ids=[f"{c['kind']}_{c['n']}" for c in DYN])
def test_oracle_dynamics(c):
    if c["kind"] == "lightvis":
        v = odyn.light_visibility(c.a("means"), c.a("depth"), c.a("cam_pos"), c.a("cam_quat"),
                                  c["half_width"], c["half_height"], c["width"], c["height"], c["bias"])
        np.testing.assert_array_equal(v, c.a("vis"))
    else:
        means = c.a("means").copy()
        quats = c.a("quats").copy()
        rows = np.flatnonzero(c.a("object_ids") == c["oid"])
        np.testing.assert_array_equal(rows, c.a("rows"))
        odyn.apply_transform(means, quats, rows, c.a("local_means"), c.a("local_rots"), c.a("q"), c.a("t"))
        np.testing.assert_array_equal(means, c.a("out_means"))
        np.testing.assert_array_equal(quats, c.a("out_quats"))
