#!/usr/bin/env python3
"""BASELINE config 1 goldens, produced by the UNMODIFIED reference.

Config 1 (BASELINE.json configs[0]): a 10k-Gaussian random field
(SURVEY §8d generator, seed 0; ground-truth model seed 1), 256x256 reference
views, 4 views per step, 100 optimizer steps, then one full snapshot
(profile 0 + zlib and profile 1), the server's baseline reset from the decoded
profile-0 snapshot (ss/server.py:481-484), one more step and one delta tick
of every attribute in DELTA_ORDER (ss/server.py:66-73, `_emit_delta`
ss/server.py:336-358).  Degrees 1 and 3.

The reference's own `splatstream.optim.step` runs every step.  Only the
per-view `backward` calls inside it are evaluated ahead of time, each by the
reference's own `backward` in a worker process (it is a pure function of the
model and the view), and handed back to `step` in the order `step` asks for
them -- so the trajectory is bit-identical to a serial run while the 4 views
of a step use 4 cores.

Written: tests/golden/config1_cases.{npz,json}.  Arrays per degree d:
  init_*      the initial model (SURVEY §8d random field)
  gts, poses  the 4 ground-truth images (reference render of the target
              model, float32) and camera poses (position, quaternion wxyz)
  losses      the 101 step losses
  s{1,10,100,101}_*  trainable attributes after that many steps
  ema100, age100     OptimizerState.grad_ema / age after step 100
  m100_*, v100_*     OptimizerState.m / .v after step 100 (the teacher-forced
                     check: the reference's step-100 state stepped once on the
                     GPU against s101_*)
  snap_p0, snap_p1   encode_snapshot payloads of the step-100 model
  base_means, base_log_scales   baselines after the reset (decoded p0)
  tick_{attr}        the DELTA_ORDER tick's payloads after step 101
  tick_base_means, tick_base_log_scales   baselines after that tick

Usage:  python tests/golden/make_config1.py [--ref /root/reference/pkg] [--degrees 1 3]
"""

from __future__ import annotations

import argparse
import json
import math
import multiprocessing as mp
import pathlib
import sys
import time

import numpy as np

HERE = pathlib.Path(__file__).resolve().parent
ROOT = HERE.parents[1]
N, W, H, VIEWS, STEPS = 10_000, 256, 256, 4, 100
CHECKPOINTS = (1, 10, 100)
FOV = 1.2
BG = np.array([0.05, 0.05, 0.08])


def random_field_arrays(n, degree, seed=0):
    """SURVEY §8d 'random field' (the same draws as paper_2604_02851_b200/synth.py)."""
    rng = np.random.default_rng(seed)
    f = (H / 2.0) / math.tan(FOV / 2.0)
    z = rng.uniform(3.0, 6.0, n)
    hy = z * (H / 2.0) / f
    hx = hy * W / H
    x = rng.uniform(-1.0, 1.0, n) * hx
    y = rng.uniform(-1.0, 1.0, n) * hy
    sig = np.exp(rng.normal(math.log(2.0), 0.5, n))
    ls = np.log(sig * z / f)[:, None] + rng.normal(0.0, 0.2, (n, 3))
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    B = (degree + 1) ** 2
    sh = np.empty((n, 3, B), np.float32)
    sh[:, :, 0] = rng.uniform(-0.5, 0.5, (n, 3))
    if B > 1:
        sh[:, :, 1:] = rng.uniform(-0.05, 0.05, (n, 3, B - 1))
    return dict(means=np.stack([x, y, z], 1).astype(np.float32), log_scales=ls.astype(np.float32),
                quaternions=q.astype(np.float32), logit_opacities=rng.uniform(-1.0, 2.0, n).astype(np.float32),
                sh_coeffs=sh, light_visibility=(rng.random(n) < 0.7).astype(np.float32),
                object_ids=np.zeros(n, np.int32))


TRAIN = ("means", "log_scales", "quaternions", "logit_opacities", "sh_coeffs")
_VIEWS = None


def _worker_init(views):
    global _VIEWS
    _VIEWS = views


def _worker_backward(args):
    from splatstream.optim import backward
    model, i = args
    return backward(model, _VIEWS[i])


def run_degree(degree):
    from splatstream.geometry import CameraIntrinsics, look_at
    from splatstream.model import GaussianModel
    from splatstream import optim as ref_optim
    from splatstream.optim import OptimizerState, ReferenceView, step
    from splatstream.protocol import PROFILE_DEFAULT, PROFILE_LOSSLESS, encode_snapshot, decode_snapshot
    from splatstream.protocol.delta import DeltaBaselines
    from splatstream.render import LightState, flat_ambient_sh, render
    from splatstream.server import DELTA_ORDER, StreamServer

    arr = random_field_arrays(N, degree)
    model = GaussianModel(**arr, active_count=N, sh_degree=degree)
    tgt = model.copy()
    rng = np.random.default_rng(1)
    tgt.sh_coeffs[:, :, 0] += rng.uniform(-0.3, 0.3, tgt.sh_coeffs[:, :, 0].shape).astype(np.float32)
    tgt.means += rng.normal(0.0, 0.01, tgt.means.shape).astype(np.float32)
    light = LightState([0.3, -1.0, 0.2], [0.6, 0.6, 0.6], flat_ambient_sh([0.35, 0.35, 0.35]))
    intr = CameraIntrinsics(width=W, height=H, fov_y=FOV, near=0.05, far=100.0)
    poses = [look_at([0.3 * math.cos(2 * math.pi * i / VIEWS), 0.3 * math.sin(2 * math.pi * i / VIEWS), 0.0],
                     [0.0, 0.0, 4.5]) for i in range(VIEWS)]
    views = [ReferenceView(p, intr, render(tgt, p, intr, light, background=BG).astype(np.float32), light, BG)
             for p in poses]
    lo = model.means.min(0).astype(np.float64) - 0.25
    hi = model.means.max(0).astype(np.float64) + 0.25
    extent = float(np.linalg.norm(hi - lo) / 2)   # as StreamServer (ss/server.py:242-247)
    state = OptimizerState(model, scene_extent=extent)

    out = {f"init_{k}": v.copy() for k, v in arr.items()}
    out.update(gts=np.stack([v.image for v in views]),
               poses=np.stack([np.concatenate([p.position, p.quaternion]) for p in poses]))

    pool = mp.get_context("fork").Pool(VIEWS, initializer=_worker_init, initargs=(views,))
    real_backward = ref_optim.backward

    def one_step():
        # evaluate the views' backward passes in parallel; step() consumes
        # them in its own order (ss/optim.py:365-372)
        results = pool.map(_worker_backward, [(model, i) for i in range(VIEWS)])
        queue = list(zip(views, results))

        def backward(m, view, index_subset=None, extent_cutoff=True):
            v, r = queue.pop(0)
            assert v is view and m is model and index_subset is None and extent_cutoff
            return r
        ref_optim.backward = backward
        try:
            return step(model, state, views)
        finally:
            ref_optim.backward = real_backward
            assert not queue

    losses = []
    t0 = time.time()
    for s in range(1, STEPS + 1):
        losses.append(one_step())
        if s in CHECKPOINTS:
            out.update({f"s{s}_{k}": model.attribute(k).copy() for k in TRAIN})
        print(f"degree {degree} step {s} loss {losses[-1]:.6f} ({time.time() - t0:.0f} s)", flush=True)
    out.update(ema100=state.grad_ema.copy(), age100=state.age.copy(),
               **{f"m100_{k}": state.m[k].copy() for k in TRAIN}, **{f"v100_{k}": state.v[k].copy() for k in TRAIN})

    # full snapshot + baseline reset from the decoded payload (ss/server.py:470-484)
    snap0 = encode_snapshot(model, PROFILE_DEFAULT)
    snap1 = encode_snapshot(model, PROFILE_LOSSLESS)
    decoded, _ = decode_snapshot(snap0)
    base = DeltaBaselines()
    base.reset_from_model(decoded, 1)
    out.update(snap_p0=np.frombuffer(snap0, np.uint8).copy(), snap_p1=np.frombuffer(snap1, np.uint8).copy(),
               base_means=base.means.copy(), base_log_scales=base.log_scales.copy())

    losses.append(one_step())
    out.update({f"s{STEPS + 1}_{k}": model.attribute(k).copy() for k in TRAIN})
    pool.close()

    # one delta tick of every attribute, through the server's own _emit_delta
    sent = []
    shim = StreamServer.__new__(StreamServer)
    shim.model, shim.baselines = model, base
    shim._send = lambda ptype, payload: sent.append(payload)
    for attr in DELTA_ORDER:
        StreamServer._emit_delta(shim, attr)
    for attr, payload in zip(DELTA_ORDER, sent):
        out[f"tick_{int(attr)}"] = np.frombuffer(payload, np.uint8).copy()
    out.update(tick_base_means=base.means.copy(), tick_base_log_scales=base.log_scales.copy(),
               losses=np.array(losses))
    meta = dict(kind="config1", degree=degree, n=N, W=W, H=H, fov=FOV, near=0.05, views=VIEWS, steps=STEPS,
                scene_extent=extent, checkpoints=list(CHECKPOINTS) + [STEPS + 1],
                tick_attrs=[int(a) for a in DELTA_ORDER][:len(sent)], bg=BG.tolist(),
                light=dict(direction=light.direction.tolist(), intensity=light.intensity.tolist(),
                           ambient=light.ambient_sh.tolist()))
    return meta, out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", default="/root/reference/pkg")
    ap.add_argument("--degrees", nargs="*", type=int, default=[1, 3])
    args = ap.parse_args()
    sys.path.insert(0, str(pathlib.Path(args.ref) / "src"))
    arrays, metas = {}, []
    for i, d in enumerate(args.degrees):
        meta, out = run_degree(d)
        metas.append(dict(meta, id=i, arrays=sorted(out)))
        arrays.update({f"c{i}_{k}": v for k, v in out.items()})
    np.savez_compressed(HERE / "config1_cases.npz", **arrays)
    (HERE / "config1_cases.json").write_text(json.dumps(metas, indent=1) + "\n")
    print("written", HERE / "config1_cases.npz")


if __name__ == "__main__":
    main()
