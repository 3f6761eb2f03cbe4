#!/usr/bin/env python3
"""Generate the golden vectors that pin the oracle and the GPU path.

Runs the UNMODIFIED reference package (read from /root/reference/pkg/src in
the build container only -- it does not exist on the GPU box) and writes:

  wire/                 the reference's own wire fixtures, regenerated with
                        pkg/scripts/make_golden_packets.py (the .bin files are
                        absent from the reference mount; the regenerated
                        manifest.json is byte-identical to the shipped one)
  codec_cases.npz/json  encode_delta / encode_snapshot inputs and payloads
  raster_cases.npz/json prepare_splats / render / backward inputs and outputs
  step_cases.npz/json   optim.step trajectories (model + OptimizerState)
  dyn_cases.npz/json    update_light_visibility / ObjectRegistry transforms
  pool_cases.npz/json   pool maintenance: GridIndex.rebuild,
                        precull, freeze_policy/freeze_range, prune,
                        OptimizerState.resize, encode_ordering, apply_mutation,
                        DeltaBaselines.apply_record
  ingest_cases.npz/json client ingestion: apply_delta onto a
                        replica + its baselines, decode_snapshot, and the
                        reference's exception (type, message) for corrupted
                        payloads

Usage:  python tests/golden/make_golden.py [--ref /root/reference/pkg] [--only NAME ...]
"""

from __future__ import annotations

import argparse
import json
import pathlib
import shutil
import subprocess
import sys

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg")
    ap.add_argument("--only", nargs="*", default=None, help="subset of: wire codec raster step dyn ingest pool engine expand objects composite")
    args = ap.parse_args()
    ref = pathlib.Path(args.ref)
    sys.path.insert(0, str(ref / "src"))
    import splatstream  # noqa: F401  (the reference)

    want = set(args.only) if args.only else {"wire", "codec", "raster", "step", "dyn", "ingest", "pool", "engine", "expand", "objects", "composite"}
    if "wire" in want:
        wire = HERE / "wire"
        if wire.exists():
            shutil.rmtree(wire)
        subprocess.run([sys.executable, str(ref / "scripts" / "make_golden_packets.py"), str(wire)], check=True)
        shipped = (ref / "tests" / "golden" / "manifest.json").read_bytes()
        assert (wire / "manifest.json").read_bytes() == shipped, "regenerated manifest differs from the shipped one"
    for name, fn in (("codec", codec_cases), ("raster", raster_cases), ("step", step_cases), ("dyn", dyn_cases),
                     ("ingest", ingest_cases), ("pool", pool_cases), ("engine", engine_cases),
                     ("expand", expand_cases), ("objects", objects_cases), ("composite", composite_cases)):
        if name in want:
            fn()
    print("golden vectors written to", HERE)


class Store:
    def __init__(self):
        self.arrays = {}
        self.cases = []

    def add(self, meta: dict, **arrays):
        i = len(self.cases)
        meta = dict(meta, id=i, arrays=sorted(arrays))
        for k, v in arrays.items():
            self.arrays[f"c{i}_{k}"] = np.asarray(v)
        self.cases.append(meta)

    def save(self, stem):
        np.savez_compressed(HERE / f"{stem}.npz", **self.arrays)
        (HERE / f"{stem}.json").write_text(json.dumps(self.cases, indent=1) + "\n")


def b2a(b: bytes):
    return np.frombuffer(b, np.uint8).copy()


def random_model(rng, n, degree, frozen=0, spread=3.0):
    from splatstream.geometry import quat_normalize
    from splatstream.model import GaussianModel
    B = (degree + 1) ** 2
    sh = np.concatenate([rng.uniform(-0.5, 0.5, (n, 3, 1)), rng.uniform(-0.1, 0.1, (n, 3, B - 1))], axis=2)
    return GaussianModel(
        means=rng.uniform(-spread, spread, (n, 3)).astype(np.float32),
        log_scales=rng.uniform(-3.5, -1.5, (n, 3)).astype(np.float32),
        quaternions=quat_normalize(rng.normal(size=(n, 4))).astype(np.float32),
        logit_opacities=rng.uniform(-2, 3, n).astype(np.float32),
        sh_coeffs=sh.astype(np.float32),
        light_visibility=(rng.random(n) > 0.4).astype(np.float32),
        object_ids=rng.integers(0, 4, n).astype(np.int32),
        active_count=n - frozen, sh_degree=degree)


def model_arrays(m):
    return dict(means=m.means, log_scales=m.log_scales, quaternions=m.quaternions,
                logit_opacities=m.logit_opacities, sh_coeffs=m.sh_coeffs,
                light_visibility=m.light_visibility, object_ids=m.object_ids)


# ------------------------------------------------------------------ codec
def codec_cases():
    from splatstream.protocol import (PROFILE_DEFAULT, PROFILE_LOSSLESS, AttributeId,
                                      QuantizationProfile, encode_delta, encode_snapshot, decode_snapshot)
    from splatstream.model import GaussianModel
    st = Store()
    rng = np.random.default_rng(1234)

    def delta(name, attr, cur, base=None, gate=None):
        arrays = dict(cur=cur)
        for comp in (0, 1):
            payload, nb = encode_delta(attr, cur, base, gating_threshold=gate, compression_id=comp)
            arrays[f"payload{comp}"] = b2a(payload)
        if base is not None:
            arrays["base"] = base
            arrays["new_base"] = nb
        st.add(dict(kind="delta", name=name, attr=int(attr), gate=gate,
                    dtype=str(np.asarray(cur).dtype)), **arrays)

    A = AttributeId
    for n in (1, 7, 40, 333, 2000):
        base = rng.uniform(-1, 1, (n, 3)).astype(np.float32)
        # dense: every row moves
        cur = (base + rng.uniform(-0.02, 0.02, base.shape)).astype(np.float32)
        delta(f"means_dense_{n}", A.MEANS, cur, base)
        delta(f"ls_dense_{n}", A.LOG_SCALES, (cur * 3 - 4).astype(np.float32), (base * 3 - 4).astype(np.float32))
        # sparse: a few rows move, some just under/over the gate
        cur = base.copy()
        mv = rng.random(n) < 0.15
        cur[mv] += rng.normal(0, 0.01, (int(mv.sum()), 3)).astype(np.float32)
        if n > 5:
            cur[3, 1] = np.float32(np.float64(base[3, 1]) + 1e-3)
            cur[4, 2] = np.float32(np.float64(base[4, 2]) + 0.99e-3)
        delta(f"means_sparse_{n}", A.MEANS, cur, base)
        delta(f"ls_sparse_{n}", A.LOG_SCALES, cur, base, gate=5e-4)
        delta(f"means_nochange_{n}", A.MEANS, base.copy(), base)
        delta(f"means_gate0_{n}", A.MEANS, cur, base, gate=0.0)
        # absolute attributes
        delta(f"quat_{n}", A.QUATERNIONS, rng.normal(0, 0.6, (n, 4)).astype(np.float32))
        delta(f"opac_{n}", A.LOGIT_OPACITIES, rng.uniform(-10, 10, n).astype(np.float32))
        delta(f"dc_{n}", A.SH_DC, rng.uniform(-5, 5, (n, 3)).astype(np.float32))
        delta(f"rest1_{n}", A.SH_REST, rng.uniform(-1.2, 1.2, (n, 3, 3)).astype(np.float32))
        delta(f"rest3_{n}", A.SH_REST, rng.uniform(-1.2, 1.2, (n, 3, 15)).astype(np.float32))
        delta(f"vis_{n}", A.LIGHT_VISIBILITY, rng.random(n).astype(np.float32))
    # large-survivor-gap varints, huge residuals, float64 input
    n = 20000
    base = rng.uniform(-1, 1, (n, 3)).astype(np.float32)
    cur = base.copy()
    cur[[0, 5, 200, 19000, 19999]] += np.float32(0.5)
    delta("means_sparse_gaps", A.MEANS, cur, base)
    cur = base.copy()
    cur[::2] += np.float32(40.0)
    delta("means_dense_huge", A.MEANS, cur, base)
    delta("means_f64_input", A.MEANS, (base[:50] + 0.01).astype(np.float64), base[:50].astype(np.float64))
    delta("opac_f64_input", A.LOGIT_OPACITIES, rng.uniform(-9, 9, 77))
    delta("means_empty", A.MEANS, np.zeros((0, 3), np.float32), np.zeros((0, 3), np.float32))
    delta("opac_empty", A.LOGIT_OPACITIES, np.zeros(0, np.float32))

    # snapshots
    for (n, deg, frozen) in ((1, 0, 0), (8, 1, 2), (64, 2, 0), (513, 3, 100), (3000, 3, 0)):
        m = random_model(rng, n, deg, frozen)
        if n == 64:
            m.means[:, 1] = np.float32(0.25)  # degenerate AABB axis
        arrays = {}
        for prof in (PROFILE_DEFAULT, PROFILE_LOSSLESS,
                     QuantizationProfile(0, 0), QuantizationProfile(1, 0)):
            payload = encode_snapshot(m, prof)
            arrays[f"payload_p{prof.profile_id}c{prof.compression_id}"] = b2a(payload)
            if prof.profile_id == 0:
                dec, _ = decode_snapshot(payload)
        st.add(dict(kind="snapshot", name=f"snap_{n}_{deg}", n=n, degree=deg, active=int(m.active_count)),
               dec_means=dec.means, dec_log_scales=dec.log_scales, **arrays, **model_arrays(m))
    m = GaussianModel.empty(2)
    payload = encode_snapshot(m, QuantizationProfile(0, 0))
    st.add(dict(kind="snapshot", name="snap_empty", n=0, degree=2, active=0),
           payload_p0c0=b2a(payload), payload_p1c0=b2a(encode_snapshot(m, QuantizationProfile(1, 0))),
           payload_p0c1=b2a(encode_snapshot(m)), payload_p1c1=b2a(encode_snapshot(m, PROFILE_LOSSLESS)),
           **model_arrays(m))
    st.save("codec_cases")


# ------------------------------------------------------------------ raster
def _pose_arrays(pose):
    return np.concatenate([pose.position, pose.quaternion])


def raster_cases():
    from splatstream.geometry import CameraIntrinsics, Pose, look_at, quat_normalize
    from splatstream.model import GaussianModel
    from splatstream.optim import ReferenceView, backward
    from splatstream.render import LightState, flat_ambient_sh, prepare_splats, render, splat_window
    st = Store()

    def light_for(rng, mode):
        direction = np.array([0.3, -1.0, 0.2]) + rng.normal(0, 0.2, 3)
        intensity = rng.uniform(0.4, 0.9, 3)
        if mode == "none":
            amb = None
        elif mode == "flat":
            amb = flat_ambient_sh(rng.uniform(0.25, 0.5, 3))
        else:
            amb = np.concatenate([flat_ambient_sh(rng.uniform(0.25, 0.5, 3)), rng.uniform(-0.1, 0.1, (3, 3))], 1)
        return LightState(direction=direction, intensity=intensity, ambient_sh=amb)

    def scene_model(rng, n, degree, W, H, fov, frozen=0, zr=(2.5, 6.0), sig=(1.2, 0.5)):
        z = rng.uniform(*zr, n)
        f = (H / 2) / np.tan(fov / 2)
        hx = z * (W / 2) / f
        hy = z * (H / 2) / f
        means = np.stack([rng.uniform(-1, 1, n) * hx * 1.1, rng.uniform(-1, 1, n) * hy * 1.1, z], -1)
        spx = np.exp(rng.normal(np.log(sig[0]), sig[1], n))
        ls = np.log(spx * z / f)[:, None] + rng.normal(0, 0.3, (n, 3))
        B = (degree + 1) ** 2
        sh = np.concatenate([rng.uniform(-0.6, 0.6, (n, 3, 1)), rng.uniform(-0.08, 0.08, (n, 3, B - 1))], 2)
        return GaussianModel(
            means=means.astype(np.float32), log_scales=ls.astype(np.float32),
            quaternions=quat_normalize(rng.normal(size=(n, 4))).astype(np.float32),
            logit_opacities=rng.uniform(-1, 2.5, n).astype(np.float32), sh_coeffs=sh.astype(np.float32),
            light_visibility=(rng.random(n) > 0.3).astype(np.float32),
            object_ids=np.zeros(n, np.int32), active_count=n - frozen, sh_degree=degree)

    def add(name, model, pose, intr, light, bg, gt_model=None, subset=None, cutoff=True, rng=None):
        prep = prepare_splats(model, pose, intr, light, subset, cutoff)
        img, T = render(model, pose, intr, light, subset, bg, return_transmittance=True, extent_cutoff=cutoff)
        if gt_model is None:
            gt = np.clip(img + rng.uniform(-0.2, 0.2, img.shape), 0, 1)
        else:
            gt = render(gt_model, pose, intr, light, None, bg, extent_cutoff=cutoff)
        view = ReferenceView(pose=pose, intrinsics=intr, image=gt.astype(np.float32), light_state=light,
                             background=np.asarray(bg, np.float64))
        L, g, img2 = backward(model, view, subset, cutoff)
        assert np.array_equal(img, img2)
        M = prep.rows.size
        wins = np.array([splat_window(prep.mu2d[i], prep.radius[i], intr.width, intr.height) for i in range(M)],
                        np.int64).reshape(M, 4)
        meta = dict(kind="raster", name=name, W=intr.width, H=intr.height, fov=float(intr.fov_y),
                    near=float(intr.near), degree=int(model.sh_degree), active=int(model.active_count),
                    cutoff=bool(cutoff), ambient=light.ambient_sh is not None, loss=L,
                    subset=subset is not None)
        arrays = dict(pose=_pose_arrays(pose), light_dir=light.direction, light_int=light.intensity,
                      bg=np.asarray(bg, np.float64), gt=view.image, image=img, T=T,
                      rows=prep.rows, order=prep.order, depth=prep.depth, mu2d=prep.mu2d,
                      Sigma2d=prep.Sigma2d, radius=prep.radius, windows=wins, color=prep.color,
                      color_pre=prep.color_pre, opacity=prep.opacity, s=prep.shade_inter["s"],
                      Sigma3d=prep.Sigma3d,
                      g_means=g.means, g_log_scales=g.log_scales, g_quaternions=g.quaternions,
                      g_logit_opacities=g.logit_opacities, g_sh_coeffs=g.sh_coeffs,
                      **model_arrays(model))
        if light.ambient_sh is not None:
            arrays["ambient"] = light.ambient_sh
        if subset is not None:
            arrays["subset"] = np.asarray(subset, np.int64)
        st.add(meta, **arrays)

    rng = np.random.default_rng(99)
    case = 0
    for degree in (0, 1, 2, 3):
        for mode in ("none", "flat", "sh1"):
            W, H, fov = (32, 24, 1.1) if case % 2 else (40, 33, 0.9)
            m = scene_model(rng, 48, degree, W, H, fov)
            tgt = m.copy()
            tgt.sh_coeffs = (tgt.sh_coeffs + rng.uniform(-0.3, 0.3, tgt.sh_coeffs.shape)).astype(np.float32)
            eye = rng.normal(0, 0.15, 3)
            pose = look_at(eye, [0.05, -0.03, 4.0])
            intr = CameraIntrinsics(width=W, height=H, fov_y=fov, near=0.05, far=100.0)
            add(f"deg{degree}_{mode}", m, pose, intr, light_for(rng, mode), (0.05, 0.05, 0.08), gt_model=tgt)
            case += 1
    # finite-difference style configuration: 16x16, cutoff disabled
    for seed in range(3):
        r2 = np.random.default_rng(500 + seed)
        m = scene_model(r2, 5, 1, 16, 16, np.pi / 2, zr=(2.5, 5.0), sig=(2.0, 0.3))
        add(f"nocutoff_{seed}", m, Pose(np.zeros(3), np.array([1.0, 0, 0, 0])),
            CameraIntrinsics(width=16, height=16, fov_y=np.pi / 2, near=0.1, far=100.0),
            light_for(r2, ("flat", "none", "sh1")[seed]), (0.0, 0.0, 0.0), cutoff=False, rng=r2)
    # frozen tail + subset + a row behind the camera
    m = scene_model(rng, 60, 2, 48, 32, 1.0, frozen=17)
    m.means[5] = [0.0, 0.0, -3.0]
    pose = look_at([0.1, 0.0, 0.0], [0.0, 0.0, 4.0])
    intr = CameraIntrinsics(width=48, height=32, fov_y=1.0, near=0.05, far=100.0)
    add("frozen_tail", m, pose, intr, light_for(rng, "flat"), (0.1, 0.2, 0.3), rng=rng)
    subset = np.sort(rng.choice(60, 35, replace=False))
    add("subset", m, pose, intr, light_for(rng, "flat"), (0.1, 0.2, 0.3), subset=subset, rng=rng)
    # capped alpha: one huge near-opaque splat plus small ones in front
    m = scene_model(rng, 6, 0, 16, 16, np.pi / 2)
    m.means[0] = [0.0, 0.0, 8.0]
    m.log_scales[0] = 6.0
    m.logit_opacities[0] = 14.0
    add("capped", m, Pose(np.zeros(3), np.array([1.0, 0, 0, 0])),
        CameraIntrinsics(width=16, height=16, fov_y=np.pi / 2, near=0.1, far=100.0),
        light_for(rng, "flat"), (0.0, 0.0, 0.0), rng=rng)
    # exact depth ties, broken by row
    m = scene_model(rng, 12, 1, 24, 24, 1.2)
    m.means[:, 2] = np.float32(4.0)
    add("depth_ties", m, Pose(np.zeros(3), np.array([1.0, 0, 0, 0])),
        CameraIntrinsics(width=24, height=24, fov_y=1.2, near=0.05, far=100.0),
        light_for(rng, "none"), (0.0, 0.0, 0.0), rng=rng)
    # dense saturated medium scene (exercises the T cutoff and many tiles)
    m = scene_model(rng, 2500, 3, 96, 64, 1.2, sig=(2.5, 0.5))
    tgt = m.copy()
    tgt.sh_coeffs = (tgt.sh_coeffs + rng.uniform(-0.3, 0.3, tgt.sh_coeffs.shape)).astype(np.float32)
    tgt.means = (tgt.means + rng.normal(0, 0.01, tgt.means.shape)).astype(np.float32)
    add("medium", m, look_at([0.2, 0.1, -0.3], [0.0, 0.0, 4.5]),
        CameraIntrinsics(width=96, height=64, fov_y=1.2, near=0.05, far=100.0),
        light_for(rng, "flat"), (0.05, 0.05, 0.08), gt_model=tgt)
    # empty model
    m = GaussianModel.empty(1)
    add("empty", m, Pose(np.zeros(3), np.array([1.0, 0, 0, 0])),
        CameraIntrinsics(width=8, height=8, fov_y=1.0), light_for(rng, "flat"), (0.2, 0.4, 0.6), rng=rng)
    st.save("raster_cases")


# ------------------------------------------------------------------ step
def step_cases():
    from splatstream.geometry import CameraIntrinsics, look_at
    from splatstream.optim import OptimizerState, ReferenceView, step
    from splatstream.render import LightState, flat_ambient_sh, render
    st = Store()
    rng = np.random.default_rng(7)
    for degree, frozen in ((1, 0), (3, 9)):
        m = random_model(rng, 40, degree, frozen, spread=1.0)
        m.means[:, 2] += np.float32(4.0)
        m.log_scales[:] = rng.uniform(-2.8, -1.8, m.log_scales.shape).astype(np.float32)
        light = LightState([0.3, -1.0, 0.2], [0.6, 0.6, 0.6], flat_ambient_sh([0.35, 0.35, 0.35]))
        intr = CameraIntrinsics(width=32, height=32, fov_y=1.2)
        poses = [look_at([0.3 * np.cos(a), 0.3 * np.sin(a), 0.0], [0, 0, 4.5]) for a in (0.0, 2.1, 4.2)]
        tgt = m.copy()
        tgt.sh_coeffs = (tgt.sh_coeffs + rng.uniform(-0.3, 0.3, tgt.sh_coeffs.shape)).astype(np.float32)
        bg = np.array([0.05, 0.05, 0.08])
        views = [ReferenceView(p, intr, render(tgt, p, intr, light, background=bg).astype(np.float32), light, bg)
                 for p in poses]
        init = model_arrays(m)
        init = {k: v.copy() for k, v in init.items()}
        state = OptimizerState(m, scene_extent=2.5)
        losses, snaps = [], {}
        for it in range(3):
            losses.append(step(m, state, views))
            for k in ("means", "log_scales", "quaternions", "logit_opacities", "sh_coeffs"):
                snaps[f"after{it}_{k}"] = m.attribute(k).copy()
        arrays = {f"init_{k}": v for k, v in init.items()}
        arrays.update(snaps)
        arrays.update({f"m_{k}": v for k, v in state.m.items()})
        arrays.update({f"v_{k}": v for k, v in state.v.items()})
        arrays.update(age=state.age, grad_ema=state.grad_ema, losses=np.array(losses),
                      poses=np.stack([_pose_arrays(p) for p in poses]),
                      gts=np.stack([v.image for v in views]), bg=bg,
                      light_dir=light.direction, light_int=light.intensity, ambient=light.ambient_sh)
        st.add(dict(kind="step", degree=degree, active=int(m.active_count), n=40, W=32, H=32, fov=1.2,
                    near=0.05, scene_extent=2.5, steps=3), **arrays)
    st.save("step_cases")


# ------------------------------------------------------------------ dynamics
def dyn_cases():
    from splatstream.geometry import OrthoCamera, look_at, quat_from_axis_angle
    from splatstream.model import ObjectRegistry
    from splatstream.render import update_light_visibility
    st = Store()
    rng = np.random.default_rng(3)
    for n in (5, 1000):
        m = random_model(rng, n, 1)
        pose = look_at([0.5, 6.0, 0.3], [0.0, 0.0, 0.0])
        cam = OrthoCamera(pose=pose, half_width=3.5, half_height=3.0, width=64, height=48, far=20.0)
        depth = rng.uniform(4.0, 9.0, (48, 64))
        mm = m.copy()
        update_light_visibility(mm, depth, cam, bias=0.02)
        st.add(dict(kind="lightvis", n=n, half_width=3.5, half_height=3.0, width=64, height=48, bias=0.02),
               means=m.means, depth=depth, cam_pos=pose.position, cam_quat=pose.quaternion,
               vis=mm.light_visibility)
        reg = ObjectRegistry()
        for oid in (1, 2, 3):
            reg.set_transform(oid, quat_from_axis_angle(rng.normal(size=3), rng.uniform(0, 3)), rng.normal(size=3))
        reg.refresh_locals(m)
        q = quat_from_axis_angle(rng.normal(size=3), 0.4)
        t = rng.normal(size=3)
        mm = m.copy()
        rows = reg.apply_transform(mm, 2, q, t)
        st.add(dict(kind="transform", n=n, oid=2), means=m.means, quats=m.quaternions, object_ids=m.object_ids,
               local_means=reg.local_means, local_rots=reg.local_rotations, q=q, t=t, rows=rows,
               out_means=mm.means, out_quats=mm.quaternions)
    st.save("dyn_cases")


# ------------------------------------------------------------------ ingestion (§8f rank 1)
def ingest_cases():
    """apply_delta / decode_snapshot on the client side, run by the reference."""
    import copy
    from splatstream.protocol import (PROFILE_DEFAULT, PROFILE_LOSSLESS, AttributeId, QuantizationProfile,
                                      encode_delta, encode_snapshot, decode_snapshot)
    from splatstream.protocol.delta import DeltaBaselines, apply_delta
    st = Store()
    rng = np.random.default_rng(4321)
    A = AttributeId

    groups = []

    def replica(n, deg, frozen):
        """A replica + drifted baselines, stored once (group) for its cases."""
        m = random_model(rng, n, deg, frozen)
        b = DeltaBaselines()
        b.reset_from_model(m, 3)
        # baselines drift from the model the way they do between ticks
        b.means = (b.means + rng.normal(0, 0.004, b.means.shape)).astype(np.float32)
        b.log_scales = (b.log_scales + rng.normal(0, 0.004, b.log_scales.shape)).astype(np.float32)
        g = len(groups)
        groups.append(g)
        st.add(dict(kind="replica", name=f"replica_{g}", group=g, active=int(m.active_count), degree=int(deg)),
               base_means=b.means, base_log_scales=b.log_scales, **model_arrays(m))
        m._golden_group = g
        return m, b

    ATTR_FIELD = {0: "means", 1: "log_scales", 2: "quaternions", 3: "logit_opacities", 4: "sh_coeffs",
                  5: "sh_coeffs", 6: "light_visibility"}

    def outcome(m, b, payload):
        mm, bb = copy.deepcopy(m), copy.deepcopy(b)
        try:
            ok = apply_delta(mm, bb, payload, 3, 3)
            return dict(ok=bool(ok)), mm, bb
        except Exception as e:  # noqa: BLE001 -- recorded for the drop-in's error parity
            return dict(error=type(e).__name__, message=str(e)), None, None

    def add_delta(name, m, b, payload, **extra):
        res, mm, bb = outcome(m, b, payload)
        arrays = dict(payload=b2a(payload))
        field_ = ATTR_FIELD.get(payload[0]) if len(payload) else None
        if mm is not None and field_ is not None:
            arrays[f"after_{field_}"] = getattr(mm, field_)
            arrays.update(after_base_means=bb.means, after_base_log_scales=bb.log_scales)
        st.add(dict(kind="delta", name=name, group=m._golden_group, field=field_, **res, **extra), **arrays)
        return res

    for (n, deg, frozen) in ((1, 0, 0), (9, 1, 2), (300, 2, 40), (1500, 3, 0), (2000, 1, 300)):
        for comp in (0, 1):
            m, b = replica(n, deg, frozen)
            a = m.active_count
            cur = (b.means[:a] + rng.uniform(-0.02, 0.02, (a, 3))).astype(np.float32)
            add_delta(f"means_dense_{n}_c{comp}", m, b, encode_delta(A.MEANS, cur, b.means[:a], compression_id=comp)[0])
            cur = b.means[:a].copy()
            mv = rng.random(a) < 0.1
            cur[mv] += rng.normal(0, 0.02, (int(mv.sum()), 3)).astype(np.float32)
            add_delta(f"means_sparse_{n}_c{comp}", m, b, encode_delta(A.MEANS, cur, b.means[:a], compression_id=comp)[0])
            cur = b.log_scales[:a].copy()
            cur[rng.random(a) < 0.3] += np.float32(0.05)
            add_delta(f"ls_sparse_{n}_c{comp}", m, b,
                      encode_delta(A.LOG_SCALES, cur, b.log_scales[:a], compression_id=comp)[0])
            add_delta(f"ls_nochange_{n}_c{comp}", m, b,
                      encode_delta(A.LOG_SCALES, b.log_scales[:a].copy(), b.log_scales[:a], compression_id=comp)[0])
            add_delta(f"quat_{n}_c{comp}", m, b,
                      encode_delta(A.QUATERNIONS, rng.normal(0, 0.6, (a, 4)).astype(np.float32), compression_id=comp)[0])
            add_delta(f"opac_{n}_c{comp}", m, b,
                      encode_delta(A.LOGIT_OPACITIES, rng.uniform(-10, 10, a).astype(np.float32), compression_id=comp)[0])
            add_delta(f"dc_{n}_c{comp}", m, b,
                      encode_delta(A.SH_DC, rng.uniform(-5, 5, (a, 3)).astype(np.float32), compression_id=comp)[0])
            if deg > 0:
                B = (deg + 1) ** 2
                add_delta(f"rest_{n}_c{comp}", m, b, encode_delta(
                    A.SH_REST, rng.uniform(-1.2, 1.2, (a, 3, B - 1)).astype(np.float32), compression_id=comp)[0])
            add_delta(f"vis_{n}_c{comp}", m, b,
                      encode_delta(A.LIGHT_VISIBILITY, rng.random(a).astype(np.float32), compression_id=comp)[0])
    # survivor gaps needing multi-byte varints, huge residuals
    m, b = replica(17000, 0, 0)
    cur = b.means.copy()
    cur[[0, 5, 200, 16500, 16999]] += np.float32(0.5)  # gaps of 1, 2 and 3 varint bytes
    add_delta("means_sparse_gaps", m, b, encode_delta(A.MEANS, cur, b.means, compression_id=0)[0])
    cur = b.means.copy()
    cur[::2] += np.float32(40.0)
    add_delta("means_dense_huge", m, b, encode_delta(A.MEANS, cur, b.means, compression_id=0)[0])
    # corrupted / inconsistent payloads: the reference's exception is the expectation
    m, b = replica(40, 2, 0)
    cur = b.means.copy()
    cur[[3, 17, 30]] += np.float32(0.01)
    good = encode_delta(A.MEANS, cur, b.means, compression_id=0)[0]   # sparse, 3 survivors
    dense = encode_delta(A.MEANS, (b.means + 0.01).astype(np.float32), b.means, compression_id=0)[0]
    opac = encode_delta(A.LOGIT_OPACITIES, rng.uniform(-3, 3, 40).astype(np.float32), compression_id=0)[0]
    quat = encode_delta(A.QUATERNIONS, rng.normal(0, 0.5, (40, 4)).astype(np.float32), compression_id=0)[0]
    import struct as _st

    def with_block(p, head_len, block):
        return p[:head_len] + _st.pack("<I", len(block)) + block

    bad = {
        "err_short": good[:5],
        "err_attr": bytes([9]) + good[1:],
        "err_mode": good[:1] + bytes([7]) + good[2:],
        "err_rows_huge": good[:4] + _st.pack("<I", (1 << 24) + 1) + good[8:],
        "err_count_mismatch": good[:4] + _st.pack("<I", 39) + good[8:],
        "err_k_gt_count": good[:16] + _st.pack("<I", 41) + good[20:],
        "err_range_nan": good[:8] + _st.pack("<ff", float("nan"), 1.0) + good[16:],
        "err_varint_truncated": with_block(good, 20, b"\x80\x80"),
        "err_varint_too_long": with_block(good, 20, b"\xff" * 12 + b"\x01" * 30),
        "err_index_range": with_block(good, 20, bytes([0, 0, 60]) + bytes(18)),
        "err_codes_truncated": with_block(good, 20, good[24:24 + 5]),
        "err_dense_codes_truncated": with_block(dense, 16, dense[20:60]),
        "err_block_oversize": with_block(opac, 8, opac[12:] + bytes(9)),
        "err_abs_truncated": with_block(quat, 8, quat[12:40]),
        "err_zlib_corrupt": good[:2] + bytes([1]) + good[3:20] + _st.pack("<I", 4) + b"\x00\x01\x02\x03",
        "err_unknown_compression": good[:2] + bytes([5]) + good[3:],
        "err_residual_absolute_attr": opac[:1] + bytes([0]) + opac[2:],
        "err_absolute_means": good[:1] + bytes([2]) + good[2:],
    }
    for name, p in bad.items():
        add_delta(name, m, b, p)
    # stale epoch: untouched, returns False
    mm, bb = copy.deepcopy(m), copy.deepcopy(b)
    assert apply_delta(mm, bb, good, 2, 3) is False

    # snapshots
    for (n, deg, frozen) in ((1, 0, 0), (9, 1, 2), (64, 2, 0), (777, 3, 100), (3000, 1, 0)):
        m = random_model(rng, n, deg, frozen)
        m.object_ids = rng.integers(0, 1 << 20, n).astype(np.int32)  # multi-byte varints
        if n == 64:
            m.means[:, 1] = np.float32(0.25)  # degenerate AABB axis
        for prof in (PROFILE_DEFAULT, PROFILE_LOSSLESS, QuantizationProfile(0, 0), QuantizationProfile(1, 0)):
            payload = encode_snapshot(m, prof)
            dec, info = decode_snapshot(payload)
            st.add(dict(kind="snapshot", name=f"snap_{n}_{deg}_p{prof.profile_id}c{prof.compression_id}",
                        active=int(dec.active_count), degree=int(dec.sh_degree)),
                   payload=b2a(payload), aabb_lo=info["aabb_lo"], aabb_hi=info["aabb_hi"],
                   **{f"dec_{k}": v for k, v in model_arrays(dec).items()})
    m = random_model(rng, 50, 1, 0)
    p0 = encode_snapshot(m, QuantizationProfile(0, 0))
    p1 = encode_snapshot(m, QuantizationProfile(1, 0))
    sbad = {
        "serr_short": p0[:30],
        "serr_truncated_block": p0[:-7],
        "serr_active": p0[:4] + _st.pack("<I", 51) + p0[8:],
        "serr_degree": p0[:8] + bytes([4]) + p0[9:],
        "serr_profile": p0[:9] + bytes([3]) + p0[10:],
        "serr_aabb_inf": p0[:12] + _st.pack("<f", float("inf")) + p0[16:],
        "serr_section": p0[:36] + _st.pack("<I", 100) + p0[40:140],
        "serr_ids_truncated": p0[:36] + _st.pack("<I", len(p0) - 40 - 20) + p0[40:-20],
        "serr_lossless_section": p1[:36] + _st.pack("<I", 400) + p1[40:440],
    }
    for name, p in sbad.items():
        try:
            decode_snapshot(p)
            res = dict(ok=True)
        except Exception as e:  # noqa: BLE001
            res = dict(error=type(e).__name__, message=str(e))
        st.add(dict(kind="snapshot_error", name=name, **res), payload=b2a(p))
    st.save("ingest_cases")


# ------------------------------------------------------------------ pool maintenance (§8f rank 2)
def pool_cases():
    import copy
    from splatstream.expansion import freeze_policy, precull, prune
    from splatstream.geometry import CameraIntrinsics, Pose
    from splatstream.model import (AppendRecord, GridIndex, PermuteRecord, PruneRecord, apply_mutation,
                                   freeze_range)
    from splatstream.optim import OptimizerState
    from splatstream.protocol.delta import DeltaBaselines
    from splatstream.protocol.packets import encode_ordering
    st = Store()
    rng = np.random.default_rng(777)

    def opt_state(m):
        o = OptimizerState(m, scene_extent=3.0)
        a = m.active_count
        for k in o.m:  # integer-valued moments: row moves are what is checked, and they compress
            o.m[k] = rng.integers(-1000, 1000, o.m[k].shape).astype(np.float64)
            o.v[k] = rng.integers(0, 1000, o.v[k].shape).astype(np.float64)
        o.age = rng.integers(0, 300, a).astype(np.int64)
        o.grad_ema = 10.0 ** rng.uniform(-7, -2, a)
        return o

    def opt_arrays(prefix, o):
        out = {f"{prefix}age": o.age, f"{prefix}grad_ema": o.grad_ema}
        for k in o.m:
            out[f"{prefix}m_{k}"] = o.m[k]
            out[f"{prefix}v_{k}"] = o.v[k]
        return out

    for (n, deg, frozen, cell) in ((1, 0, 0, 2.0), (50, 1, 10, 1.5), (3000, 2, 400, 1.0), (8000, 1, 900, 0.7)):
        m = random_model(rng, n, deg, frozen, spread=4.0)
        m.logit_opacities[:] = rng.uniform(-6, 3, n).astype(np.float32)  # some below the 0.01 floor
        o = opt_state(m)
        b = DeltaBaselines()
        b.reset_from_model(m, 1)
        base_arrays = dict(**model_arrays(m), **opt_arrays("opt_", o), base_means=b.means, base_log_scales=b.log_scales)
        # grid + precull
        grid = GridIndex(cell_size=cell, origin=(0.1, -0.2, 0.3))
        grid.rebuild(m)
        keys = np.array(list(grid.cell_map.keys()), np.int64).reshape(-1, 3)
        lens = np.array([len(v) for v in grid.cell_map.values()], np.int64)
        rows = np.concatenate([np.array(v, np.int64) for v in grid.cell_map.values()]) if n else np.zeros(0, np.int64)
        intr = CameraIntrinsics(width=96, height=64, fov_y=np.deg2rad(60), near=0.2, far=9.0)
        poses = [Pose(np.array([0.0, 0.0, -6.0]), np.array([1.0, 0.0, 0.0, 0.0])),
                 Pose(np.array([5.0, 1.0, 0.0]), np.array([0.7071, 0.0, -0.7071, 0.0]))]
        keep = precull(m, grid, poses, intr)
        depth = [rng.uniform(2.0, 9.0, (64, 96)), rng.uniform(2.0, 9.0, (64, 96))]
        keep_d = precull(m, grid, poses, intr, depth)
        pose_arr = np.array([np.concatenate([p.position, p.quaternion]) for p in poses])
        # freeze
        frz = freeze_policy(m, o, age_threshold=120, grad_threshold=3e-4)
        mf, of, bf = copy.deepcopy(m), copy.deepcopy(o), copy.deepcopy(b)
        prec = freeze_range(mf, frz)
        if prec is not None:
            of.resize(prec)
            bf.apply_record(prec)
        # prune
        mp, op_, bp = copy.deepcopy(m), copy.deepcopy(o), copy.deepcopy(b)
        removed, rrec = prune(mp, opacity_floor=0.01)
        if rrec is not None:
            op_.resize(rrec)
            bp.apply_record(rrec)
        # append (placeholders on the client) + ordering packet over all three records
        ids = rng.integers(0, 5, 7).astype(np.int32)
        arec = AppendRecord(insert_at=int(m.active_count), count=7, object_ids=ids,
                            new_active_count=int(m.active_count) + 7)
        recs = [r for r in (prec,) if r is not None]
        packet = encode_ordering(recs + [arec] + ([rrec] if rrec is not None else []))
        ma = copy.deepcopy(m)
        apply_mutation(ma, arec)
        ba = copy.deepcopy(b)
        ba.apply_record(arec)
        oa = copy.deepcopy(o)
        oa.resize(arec)
        arrays = dict(base_arrays, cell_keys=keys, cell_lens=lens, cell_rows=rows, precull=keep, precull_depth=keep_d,
                      depth0=depth[0], depth1=depth[1], poses=pose_arr, freeze=frz, removed=removed,
                      append_ids=ids, packet=b2a(packet),
                      **{f"frozen_{k}": v for k, v in model_arrays(mf).items()}, **opt_arrays("frozen_opt_", of),
                      frozen_base_means=bf.means, frozen_base_log_scales=bf.log_scales,
                      **{f"pruned_{k}": v for k, v in model_arrays(mp).items()}, **opt_arrays("pruned_opt_", op_),
                      pruned_base_means=bp.means, pruned_base_log_scales=bp.log_scales,
                      **{f"appended_{k}": v for k, v in model_arrays(ma).items()}, **opt_arrays("appended_opt_", oa),
                      appended_base_means=ba.means, appended_base_log_scales=ba.log_scales)
        if prec is not None:
            arrays["permutation"] = prec.permutation
        st.add(dict(kind="pool", name=f"pool_{n}_{deg}", n=n, degree=deg, active=int(m.active_count), cell=cell,
                    origin=[0.1, -0.2, 0.3], width=96, height=64, fov_y=float(np.deg2rad(60)), near=0.2, far=9.0,
                    frozen_active=int(mf.active_count), pruned_active=int(mp.active_count),
                    has_permute=prec is not None, has_prune=rrec is not None), **arrays)
    st.save("pool_cases")



ENGINE_SCENES = {
    "floor_ball_box": {
        "background": [0.05, 0.05, 0.08],
        "light": {"direction": [-0.4, -1.0, 0.3], "intensity": [0.8, 0.8, 0.8], "ambient": [0.2, 0.2, 0.2]},
        "objects": [
            {"id": 0, "shape": {"kind": "plane", "point": [0, 0, 0], "normal": [0, 1, 0], "extent": [4.0, 4.0]},
             "albedo": {"kind": "checker", "colors": [[0.9, 0.9, 0.9], [0.2, 0.25, 0.35]], "scale": 1.0}},
            {"id": 1, "shape": {"kind": "sphere", "center": [0, 0.5, 0], "radius": 0.5},
             "albedo": {"kind": "solid", "color": [0.8, 0.2, 0.15]},
             "animation": {"kind": "bounce", "height": 1.0, "period": 2.0}},
            {"id": 2, "shape": {"kind": "box", "center": [1.2, 0.4, -0.6], "half_extents": [0.3, 0.4, 0.25]},
             "albedo": {"kind": "checker", "colors": [[0.1, 0.7, 0.2], [0.9, 0.8, 0.1]], "scale": 0.25},
             "animation": {"kind": "rotate", "axis": [0.2, 1.0, 0.1], "deg_per_s": 40.0, "anchor": [1.2, 0.4, -0.6]}},
            {"id": 0, "shape": {"kind": "box", "center": [-1.3, 0.3, 0.9], "half_extents": [0.3, 0.3, 0.3]},
             "albedo": {"kind": "solid", "color": [0.3, 0.4, 0.9]}},
        ],
    },
    "walls": {
        "background": [0.3, 0.1, 0.2],
        "light": {"direction": [0.5, -0.7, -0.2], "intensity": [1.0, 0.9, 0.8], "ambient": [0.15, 0.2, 0.25]},
        "objects": [
            {"id": 0, "shape": {"kind": "plane", "point": [0, -0.5, 0], "normal": [0.0, 1.0, 0.05]},
             "albedo": {"kind": "checker", "colors": [[0.8, 0.8, 0.7], [0.3, 0.3, 0.3]], "scale": 0.5}},
            {"id": 0, "shape": {"kind": "plane", "point": [0, 0, 3], "normal": [0.1, 0, -1], "extent": [2.0, 1.5]},
             "albedo": {"kind": "solid", "color": [0.6, 0.5, 0.4]}},
            {"id": 3, "shape": {"kind": "sphere", "center": [0.4, 0.2, 1.0], "radius": 0.45},
             "albedo": {"kind": "checker", "colors": [[1.0, 0.2, 0.2], [0.2, 0.2, 1.0]], "scale": 0.2},
             "animation": {"kind": "oscillate", "axis": [1, 0, 0], "amplitude": 0.3, "period": 1.5}},
        ],
    },
}


def engine_cases():
    """The reference engine (ref engine.py) on scenes built by its own
    scene_from_dict: ground truth, capture buffers, render depth, ortho depth.
    Poses are stored as (position, rotation matrix) so the device sees the
    reference's exact camera frame."""
    from splatstream.engine import (build_light_camera, capture_input_buffers, render_depth, render_ground_truth,
                                    render_ortho_depth)
    from splatstream.geometry import CameraIntrinsics, look_at
    from splatstream.scene import scene_from_dict
    st = Store()
    cams = [((2.5, 2.5, 2.5), (0, 0.3, 0), 64, 48, 1.2), ((0.3, 1.2, -3.0), (0, 0.4, 0.5), 40, 40, 0.9),
            ((-2.0, 3.5, 1.0), (0.2, 0, 0.1), 33, 27, 1.4)]
    for name, sd in ENGINE_SCENES.items():
        scene = scene_from_dict(sd)
        for time in (None, 0.7):
            tfs = scene.transforms_at(time) if time is not None else None
            tf_arr = np.array([[oid] + list(q) + list(t) for oid, (q, t) in sorted(tfs.items())]) if tfs else \
                np.zeros((0, 8))
            for ci, (eye, tgt, w, h, fov) in enumerate(cams):
                pose = look_at(np.array(eye, float), np.array(tgt, float))
                intr = CameraIntrinsics(width=w, height=h, fov_y=fov, near=0.05, far=30.0)
                gt = render_ground_truth(scene, pose, intr, transforms=tfs)
                b = capture_input_buffers(scene, pose, intr, transforms=tfs)
                dep = render_depth(scene, pose, intr, transforms=tfs)
                st.add(dict(kind="pinhole", name=f"{name}_t{time}_c{ci}", scene=sd, width=w, height=h, fov_y=fov,
                            near=0.05, far=30.0),
                       transforms=tf_arr, position=pose.position, R=pose.rotation(), gt=gt, world_pos=b.world_pos,
                       valid=b.valid, normal=b.normal, albedo=b.albedo, shaded=b.shaded, object_id=b.object_id,
                       depth=b.depth, footprint=b.footprint, lit=b.lit, render_depth=dep)
            lo, hi = scene.aabb(tfs)
            lc = build_light_camera(lo, hi, scene.light.direction, resolution=32)
            od = render_ortho_depth(scene, lc, transforms=tfs)
            st.add(dict(kind="ortho", name=f"{name}_t{time}_light", scene=sd, width=lc.width, height=lc.height,
                        half_width=lc.half_width, half_height=lc.half_height, far=lc.far),
                   transforms=tf_arr, position=lc.pose.position, R=lc.pose.rotation(), ortho_depth=od)
    # trace (engine.py:88) on arbitrary rays: per-ray directions, and shadow-style rays
    # sharing one broadcast direction (light_occluded, engine.py:130-137)
    from splatstream.engine import light_occluded, trace
    rng = np.random.default_rng(99)
    for name, sd in ENGINE_SCENES.items():
        scene = scene_from_dict(sd)
        tfs = scene.transforms_at(0.7)
        tf_arr = np.array([[oid] + list(q) + list(t) for oid, (q, t) in sorted(tfs.items())])
        org = rng.uniform(-3, 3, (500, 3)) + np.array([0, 2.5, 0])
        tgt = rng.uniform(-1.5, 1.5, (500, 3)) * np.array([1, 0.5, 1])
        dirs = tgt - org
        dirs /= np.linalg.norm(dirs, axis=-1, keepdims=True)
        h = trace(scene, org, dirs, tfs)
        pts = org[:200] * np.array([1, 0, 1])
        nrm = np.tile([0.0, 1.0, 0.0], (200, 1))
        occ = light_occluded(scene, pts, nrm, scene.light, tfs)
        st.add(dict(kind="trace", name=f"{name}_trace", scene=sd), transforms=tf_arr, origins=org, dirs=dirs,
               t=h.t, object_index=h.object_index, world_point=h.world_point, normal=h.normal, albedo=h.albedo,
               occ_points=pts, occ_normals=nrm, occluded=occ)
    st.save("engine_cases")


def expand_cases():
    """cull_input_samples + init_gaussians, run by the reference on its own
    capture buffers (dome rigs; one rig with a duplicated camera for ties)."""
    from splatstream.engine import build_dome_rig, capture_input_buffers, cull_input_samples
    from splatstream.expansion import init_gaussians
    from splatstream.scene import scene_from_dict
    st = Store()
    chans = ("world_pos", "valid", "normal", "albedo", "object_id", "footprint", "lit")
    rigs = [("floor_ball_box", (0, 0.3, 0), 0.4, 5, 2.8, 40, 32, None),
            ("walls", (0.2, 0.0, 1.2), 1.1, 3, 2.0, 36, 30, None),
            ("floor_ball_box", (0.5, 0.2, -0.2), 2.0, 3, 3.0, 32, 32, 1)]  # camera 1 duplicated as camera 3
    for name, centre, heading, ncam, radius, w, h, dup in rigs:
        scene = scene_from_dict(ENGINE_SCENES[name])
        poses, intr = build_dome_rig(np.array(centre, float), heading, ncam, radius, width=w, height=h, fov_y=1.3)
        if dup is not None:
            poses = list(poses) + [poses[dup]]
        bufs = [capture_input_buffers(scene, p, intr) for p in poses]
        sb = cull_input_samples(bufs)
        arrays = {}
        for ci, b in enumerate(bufs):
            for ch in chans:
                arrays[f"cam{ci}_{ch}"] = getattr(b, ch)
            arrays[f"cam{ci}_position"] = b.pose.position
        for k in ("positions", "normals", "albedo", "object_ids", "footprints", "lit", "camera_indices"):
            arrays[f"out_{k}"] = getattr(sb, k)
        for deg in (0, 1):
            g = init_gaussians(sb, sh_degree=deg)
            for k in ("means", "log_scales", "quaternions", "logit_opacities", "sh_coeffs", "light_visibility",
                      "object_ids"):
                arrays[f"init{deg}_{k}"] = getattr(g, k)
        st.add(dict(kind="expand", name=f"{name}_{ncam}cams" + ("_dup" if dup is not None else ""), n_cams=len(bufs),
                    kept=int(sb.count)), **arrays)
    st.save("expand_cases")


def objects_cases():
    """ObjectRegistry (ref model.py:326-404) through a server-like sequence:
    refresh all, move object 1, optimizer-style edits of object 2 rows and a
    refresh of just those rows, a row permutation, then move object 2."""
    from splatstream.geometry import quat_from_axis_angle
    from splatstream.model import ObjectRegistry, PermuteRecord, apply_mutation
    st = Store()
    rng = np.random.default_rng(2024)
    for n, deg in ((3000, 0), (20000, 1)):
        m = random_model(rng, n, deg)
        m.object_ids[:] = rng.choice([0, 0, 1, 2], n).astype(np.int32)
        reg = ObjectRegistry()
        reg.set_transform(1, quat_from_axis_angle([0, 1, 0], 0.3), [0.5, 0.0, -0.2])
        reg.set_transform(2, quat_from_axis_angle([1, 0.2, 0], -0.7), [0.0, 0.4, 0.1])
        arrays = {f"init_{k}": np.array(v, copy=True) for k, v in model_arrays(m).items()}
        reg.refresh_locals(m)
        arrays.update(lm0=reg.local_means.copy(), lr0=reg.local_rotations.copy())
        q1, t1 = quat_from_axis_angle([0.3, 1, 0], 0.9), np.array([0.2, -0.1, 0.7])
        rows1 = reg.apply_transform(m, 1, q1, t1)
        arrays.update(q1=q1, t1=t1, rows1=rows1, means1=m.means.copy(), quats1=m.quaternions.copy())
        sub = np.sort(rng.choice(n, n // 5, replace=False))
        m.means[sub] += rng.normal(0, 1e-2, (len(sub), 3)).astype(np.float32)
        arrays.update(sub=sub, means_edit=m.means.copy())
        reg.refresh_locals(m, sub)
        arrays.update(lm2=reg.local_means.copy(), lr2=reg.local_rotations.copy())
        perm = rng.permutation(n)
        rec = PermuteRecord(perm, m.active_count)
        apply_mutation(m, rec)
        reg.resize(rec)
        q2, t2 = quat_from_axis_angle([0, 0, 1], 1.3), np.array([-0.3, 0.2, 0.0])
        rows2 = reg.apply_transform(m, 2, q2, t2)
        arrays.update(perm=perm, q2=q2, t2=t2, rows2=rows2, means3=m.means.copy(), quats3=m.quaternions.copy(),
                      lm3=reg.local_means.copy(), lr3=reg.local_rotations.copy())
        st.add(dict(kind="objects", name=f"objects_{n}_deg{deg}", n=n, degree=deg, active=int(m.active_count)),
               **arrays)
    st.save("objects_cases")


def composite_cases():
    """render.composite (ref render.py:317-336) on the reference's own
    PreparedSplats, as prepared and after edits (opacity, colour, draw order,
    an infinite radius), so the device blend is checked on arbitrary inputs."""
    from splatstream.geometry import CameraIntrinsics, look_at
    from splatstream.render import LightState, composite, prepare_splats
    st = Store()
    rng = np.random.default_rng(31)
    for n, deg, W, H in ((2000, 1, 96, 64), (6000, 3, 130, 70)):
        m = random_model(rng, n, deg, spread=1.5)
        m.means[:, 2] += 4.0
        pose = look_at(np.array([0.2, -0.1, -1.0]), np.array([0.0, 0.0, 4.0]))
        intr = CameraIntrinsics(width=W, height=H, fov_y=1.0, near=0.05)
        light = LightState(direction=np.array([-0.3, -1.0, 0.2]), intensity=np.array([0.8, 0.8, 0.8]))
        prep = prepare_splats(m, pose, intr, light)
        for variant in ("as_prepared", "edited"):
            if variant == "edited":
                prep.opacity = prep.opacity * 0.5
                prep.color = prep.color[:, ::-1].copy()
                prep.order = prep.order[::-1].copy()
                prep.radius = prep.radius.copy()
                prep.radius[prep.order[:3]] = np.inf
            img, T = composite(prep, intr, np.array([0.1, 0.2, 0.3]))
            st.add(dict(kind="composite", name=f"composite_{n}_{variant}", W=W, H=H),
                   order=prep.order, mu2d=prep.mu2d, radius=prep.radius, inv2d=prep.inv2d, opacity=prep.opacity,
                   color=prep.color, img=img, T=T)
    st.save("composite_cases")

if __name__ == "__main__":
    main()
