#!/usr/bin/env python3
"""Throughput of the splatstream server hot path on B200.

Workload (BASELINE.json config 3, the one the metric is quoted on):
1M Gaussians, SH degree 3, 8 reference views of 1920x1080 per optimizer
step, sharded over the ranks (views r, r+N, ...), gradients summed with one
NCCL all-reduce, fp64-moment Adam on every rank; rank 0 then encodes the
per-frame delta tick (DEFAULT_DELTA_PERIODS of ref server.py:57-64,
compression_id 0).  A "step" is one optimizer step over the 8 views plus
that delta tick.

  python bench.py [--gpus N --steps K --warmup W]          # our arm
  python bench.py --impl reference [--steps K --warmup W]  # CPU reference arm

Metric: optimize views/s (views per step x steps/s, ref cli.py:370-372);
whole-job aggregate over ranks.  `e2e` is the same metric through the
public API (optim.step + protocol.DeltaTicker, payloads read back to host) with the step's ground-truth
images copied from pinned host memory every step and the loss and delta
payload bytes read back.  The reference arm times the CPU oracle port of the
reference algorithm (oracle/, numpy float64) on the host's cores.
"""

from __future__ import annotations

import argparse
import gc
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "3DGS optimize views/sec at 1M Gaussians 1080p; delta-encode Gaussians/sec"
DELTA_ORDER = (0, 1, 2, 3, 4, 5)  # means, log_scales, quaternions, opacities, sh_dc, sh_rest
DELTA_PERIODS = {0: 1, 1: 1, 2: 10, 3: 1, 4: 1, 5: 30}
CROP = 12  # CPU sample: a centre crop of 1/CROP^2 of every view


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--views", type=int, default=8)
    ap.add_argument("--width", type=int, default=1920)
    ap.add_argument("--height", type=int, default=1080)
    ap.add_argument("--degree", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--atomics", action="store_true", help="with --step-only: also time the atomics mode")
    ap.add_argument("--step-only", action="store_true",
                    help="profiling: only the timed optimize steps (no encoder / pool / engine / e2e records)")
    return ap.parse_args()


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi polled every 50 ms on a reader thread; each sample is stamped
    with the host clock so only the samples inside the timed window count."""
    FIELDS = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.samples = []
        self.thread = None

    def start(self):
        import threading
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return

        def read():
            for line in self.proc.stdout:
                self.samples.append((time.time(), line))
        self.thread = threading.Thread(target=read, daemon=True)
        self.thread.start()

    def wait_first(self, timeout=5.0):
        t = time.time() + timeout
        while self.proc is not None and not self.samples and time.time() < t:
            time.sleep(0.02)

    def stop(self, t_begin, t_end):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread is not None:
            self.thread.join(timeout=5)
        sm, mx, reasons = [], 0.0, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        import datetime
        for ts, line in self.samples:
            p = [x.strip() for x in line.split(",")]
            if len(p) < 10:
                continue
            try:  # nvidia-smi's own sample time (stdout may arrive in bursts)
                ts = datetime.datetime.strptime(p[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
            except ValueError:
                pass
            if not (t_begin <= ts <= t_end):
                continue
            try:
                sm.append(float(p[2]))
                mx = max(mx, float(p[3]))
            except ValueError:
                continue
            for name, v in zip(names, p[6:10]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm),
                "window_s": round(t_end - t_begin, 3)}


# ---------------------------------------------------------------- CPU oracle sample
def crop_camera(cam, crop=CROP, k=0, per_view=1):
    """The k-th of `per_view` crops of 1/crop^2 of the frame, side by side
    around the centre; returns (camera, frame px / sampled px of the view)."""
    w, h = cam["W"] // crop, cam["H"] // crop
    x0 = (cam["W"] - per_view * w) // 2 + k * w
    y0 = (cam["H"] - h) // 2
    c = dict(cam)
    c.update(W=w, H=h, cx=cam["cx"] - x0, cy=cam["cy"] - y0)
    return c, (cam["W"] * cam["H"]) / (per_view * w * h)


def cpu_sample_setup(model, tgt, poses, intr, light_state, crop=CROP, per_view=1):
    """Per view and crop: crop camera, rows whose window meets the crop, oracle GT."""
    from oracle import raster as orr
    light = dict(direction=light_state.direction, intensity=light_state.intensity, ambient=light_state.ambient_sh)
    jobs = []
    for pose in poses:
        cam = orr.camera(pose, intr)
        for k in range(per_view):
            ccam, factor = crop_camera(cam, crop, k, per_view)
            prep = orr.prepare(model, ccam, light, None, True)
            r = prep["rect"]
            rows = prep["rows"][(r[:, 0] < r[:, 1]) & (r[:, 2] < r[:, 3])]
            gt, _ = orr.render(tgt, ccam, light, (0.05, 0.05, 0.08), rows, True)
            jobs.append((ccam, rows, gt))
    return light, jobs, factor


_POOL_STATE = {}


def _pool_init(model, light):
    _POOL_STATE["model"] = model
    _POOL_STATE["light"] = light


def _pool_backward(job):
    from oracle import raster as orr
    ccam, rows, gt = job
    t0 = time.perf_counter()
    orr.backward(_POOL_STATE["model"], ccam, _POOL_STATE["light"], gt, (0.05, 0.05, 0.08), rows, True)
    return time.perf_counter() - t0


def oracle_delta_tick(model, base_means, base_ls, tick):
    from oracle import codec as oc
    a = model.active_count
    rows = 0
    for attr in DELTA_ORDER:
        if tick % DELTA_PERIODS[attr]:
            continue
        if attr == 0:
            oc.delta_payload(0, model.means[:a], base_means[:a], None, 0)
        elif attr == 1:
            oc.delta_payload(1, model.log_scales[:a], base_ls[:a], None, 0)
        elif attr == 2:
            oc.delta_payload(2, model.quaternions[:a], None, None, 0)
        elif attr == 3:
            oc.delta_payload(3, model.logit_opacities[:a], None, None, 0)
        elif attr == 4:
            oc.delta_payload(4, model.sh_coeffs[:a, :, 0], None, None, 0)
        else:
            oc.delta_payload(5, model.sh_coeffs[:a, :, 1:], None, None, 0)
        rows += a
    return rows


def build_workload(args):
    from paper_2604_02851_b200 import synth
    model = synth.random_field(args.n, args.degree, args.width, args.height, seed=0)
    tgt = synth.target_model(model, seed=1)
    poses = synth.ring_poses(args.views)
    intr = synth.intrinsics(args.width, args.height)
    return model, tgt, poses, intr, synth.light()


def run_reference(args):
    """CPU arm: the oracle port of the reference algorithm on all host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import multiprocessing as mp
    model, tgt, poses, intr, light_state = build_workload(args)
    cores = os.cpu_count() or 1
    per_view = max(1, cores // len(poses))  # crops per view so every core has a job
    light, jobs, factor = cpu_sample_setup(model, tgt, poses, intr, light_state, per_view=per_view)
    procs = min(cores, len(jobs))
    base_m = model.means.copy()
    base_l = model.log_scales.copy()
    ctx = mp.get_context("fork")
    # Adam (ref optim.py:374-406) on a row sample, time x (active rows / sample rows)
    from oracle import adam as oadam
    B = (model.sh_degree + 1) ** 2
    a = int(model.active_count)
    ra = min(a, 100_000)
    sample_model = GaussianModelSlice(model, ra)
    ast = oadam.AdamState(ra, B)
    rng = np.random.default_rng(0)
    grads = dict(means=rng.normal(0, 1e-3, (ra, 3)), log_scales=rng.normal(0, 1e-3, (ra, 3)),
                 quaternions=rng.normal(0, 1e-3, (ra, 4)), logit_opacities=rng.normal(0, 1e-3, ra),
                 sh_coeffs=rng.normal(0, 1e-3, (ra, 3, B)))
    times = []
    walls = []
    with ctx.Pool(procs, initializer=_pool_init, initargs=(model, light)) as pool:
        for i in range(args.warmup + args.steps):
            w0 = time.perf_counter()
            t0 = time.perf_counter()
            view_times = pool.map(_pool_backward, jobs)
            t_views = time.perf_counter() - t0
            t1 = time.perf_counter()
            oadam.apply(sample_model, ast, grads, len(poses))
            t_adam = time.perf_counter() - t1
            t1 = time.perf_counter()
            oracle_delta_tick(model, base_m, base_l, i)
            t_delta = time.perf_counter() - t1
            if i >= args.warmup:
                times.append((t_views, t_adam, t_delta))
                walls.append(time.perf_counter() - w0)
    t_step = float(np.mean([tv * factor + ta * (a / ra) + td for tv, ta, td in times]))
    value = len(poses) / t_step
    sample = (f"oracle numpy float64 backward of each of the {len(poses)} views on {per_view} crop(s) of "
              f"{intr.width // CROP}x{intr.height // CROP} px (1/{factor:.0f} of the frame per view; only rows whose "
              f"window meets the crop), {procs} processes in parallel, time x{factor:.0f} (extrapolated to the full "
              f"frame) + Adam on {ra} of the {a} rows, time x{a / ra:.0f} + the full-size {args.n}-row delta tick "
              f"(raw); measured wall per sampled step {np.mean(walls) * 1e3:.0f} ms, ms_per_step is the extrapolation")
    out = {"metric": METRIC, "value": value, "unit": "views/s", "n_gpus": args.gpus, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": t_step * 1e3, "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
           "config": workload_config(args),
           "cpu_baseline": {"value": value, "unit": "views/s", "cores": procs, "kind": "port", "sample": sample},
           "e2e": {"value": value, "unit": "views/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


class GaussianModelSlice:
    """The first `rows` rows of a host model as an active-only model (the
    reference arm's Adam sample)."""

    def __init__(self, model, rows):
        for k in ("means", "log_scales", "quaternions", "logit_opacities", "sh_coeffs"):
            setattr(self, k, np.array(getattr(model, k)[:rows]))
        self.active_count = rows
        self.sh_degree = model.sh_degree


def workload_config(args):
    return {"workload": (f"config3: {args.n} Gaussians SH{args.degree}, {args.views} reference views "
                         f"{args.width}x{args.height} per optimizer step sharded over the GPUs + per-frame delta "
                         "tick (raw)"),
            "gaussians": args.n, "views_per_step": args.views, "resolution": f"{args.width}x{args.height}",
            "sh_degree": args.degree, "l2": "no flush: per-step working set (244 MB model, 944 MB Adam moments, "
                                            "~190 MB partials, 199 MB GT) exceeds the 126 MB L2",
            "view_lanes": _view_lanes(),
            "kernel_timing": "kernel_ms_per_step / roofline / gpu_launches from a second pass of the same steps "
                             "with the view lanes on one stream (each kernel timed alone)"}


def _view_lanes():
    from paper_2604_02851_b200 import optim
    return optim.VIEW_LANES


# ---------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2604_02851_b200 import _lib
    from paper_2604_02851_b200 import optim as optim_mod
    from paper_2604_02851_b200.model import DeviceModel
    from paper_2604_02851_b200.optim import OptimizerState, ReferenceView, StepWorkspace, step
    from paper_2604_02851_b200.protocol import DeltaTicker, PayloadBuffer, encode_snapshot_device
    from paper_2604_02851_b200.render import render_device

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # functional check of the multi-rank orchestration on a one-GPU box only:
    # SS_BENCH_BACKEND=gloo SS_BENCH_SAME_DEVICE=1 puts every rank on cuda:0
    # with host-staged collectives (no rank's kernels wait on another's);
    # its numbers measure nothing
    backend = os.environ.get("SS_BENCH_BACKEND", "nccl")
    if os.environ.get("SS_BENCH_SAME_DEVICE") == "1":
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
        pg = dist.group.WORLD

    model_h, tgt_h, poses, intr, light = build_workload(args)
    dm = DeviceModel.from_host(model_h, local)
    tgt = DeviceModel.from_host(tgt_h, local)
    mine = list(range(rank, args.views, world))
    bg = np.array([0.05, 0.05, 0.08])
    gts = [render_device(tgt, poses[v], intr, light, background=bg) for v in mine]
    del tgt
    # every rank passes all the step's views (step() shards them); a view
    # rendered elsewhere only needs its camera here: a stride-0 placeholder image
    placeholder = torch.zeros((1, 1, 1), dtype=torch.float32, device=dev).expand(intr.height, intr.width, 3)
    img_of = dict(zip(mine, gts))
    views = [ReferenceView(poses[v], intr, img_of.get(v, placeholder), light, bg) for v in range(args.views)]
    lo, hi = model_h.means.min(0), model_h.means.max(0)
    state = OptimizerState(dm, scene_extent=float(np.linalg.norm(hi - lo) / 2), device=dev, process_group=pg)
    ws = StepWorkspace(dm)
    a = dm.active_count

    def solo_state():
        """Rank 0's single-GPU records run without the other ranks: their own state."""
        if pg is None:
            return state
        return OptimizerState(dm, scene_extent=state.scene_extent, device=dev)
    # delta baselines from the decoded snapshot (server.py:481-484), computed on device
    base_m = torch.empty((dm.count, 3), dtype=torch.float32, device=dev)
    base_l = torch.empty((dm.count, 3), dtype=torch.float32, device=dev)
    encode_snapshot_device(dm, 0, None, base_m, base_l)
    bufs = {attr: PayloadBuffer(1 << 20, dev) for attr in DELTA_ORDER}

    baselines = {0: base_m[:a], 1: base_l[:a]}
    ticker = DeltaTicker(dm, baselines, bufs)
    pend = [None]  # e2e: the previous tick's payload readback in flight

    def delta_tick(tick, device_only=True):
        """Rank 0 encodes the attributes due this tick (server.py:488-493)."""
        if rank != 0:
            return 0, 0
        due = [attr for attr in DELTA_ORDER if tick % DELTA_PERIODS[attr] == 0]
        if device_only:  # one batched library call, payloads stay in HBM
            return ticker(due), 0
        # public API: batched encode, device CRC of each payload, then every
        # TENSOR_DELTA frame (envelope + payload + CRC) assembled in pinned host memory
        ticker(due)
        pending = ticker.read_async(due, frame_epoch=1)  # collected after the next step is queued (one tick of latency)
        done, pend[0] = pend[0], pending
        return a * len(due), (sum(len(p) for p in done.result(copy=False)) if done is not None else 0)

    c = _lib.ctx(local)
    fp32_peak = ctypes_peak(c)

    def one_step(i):
        step(dm, state, views, workspace=ws, sync_loss=False)
        return delta_tick(i)

    clocks = ClockSampler(local)
    clocks.start()
    for i in range(args.warmup):
        one_step(i)
    clocks.wait_first()
    torch.cuda.synchronize()
    if pg is not None:
        dist.barrier()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    if pg is not None:
        dist.barrier()
    w0 = time.time()
    t0.record()
    delta_rows = 0
    for i in range(args.steps):
        r, _ = one_step(args.warmup + i)
        delta_rows += r
    t1.record()
    torch.cuda.synchronize()
    if pg is not None:
        dist.barrier()
    w1 = time.time()
    ms = t0.elapsed_time(t1)
    clock_rec = clocks.stop(w0, w1)
    ms_t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if pg is not None:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())
    ms_per_step = ms / args.steps
    value = args.views * args.steps / (ms / 1e3)

    # ---- e2e through the public API with host buffers, right after the
    # device-resident region (the same model state: every later record trains
    # the model further, and its pair counts drift)
    e2e = None
    if not args.no_e2e and not args.step_only:
        host_gt = [g.cpu().pin_memory() for g in gts]
        himg = dict(zip(mine, host_gt))
        hviews = [ReferenceView(poses[v], intr, himg.get(v, placeholder), light, bg) for v in range(args.views)]
        h2d = sum(int(g.numel()) * 4 for g in host_gt)
        d2h = 0
        for i in range(2):
            step(dm, state, hviews, workspace=ws)
            delta_tick(i, device_only=False)
        if pend[0] is not None:
            pend[0].result(copy=False)
            pend[0] = None
        torch.cuda.synchronize()
        if pg is not None:
            dist.barrier()
        # The loss is read back like the payloads: an async copy into pinned
        # memory collected one step later (the last one inside the region), so
        # the host never stalls the stream between steps.  (Allocated before
        # the timed region: a pinned allocation can stall the device.)
        loss_h = torch.zeros(2, dtype=torch.float64).pin_memory()
        loss_ev = [torch.cuda.Event(), torch.cuda.Event()]
        losses = []
        gc.collect()
        gc.disable()  # no collector pauses inside the timed region (re-enabled right after)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(args.steps):
            lt = step(dm, state, hviews, workspace=ws, sync_loss=False)
            loss_h[i % 2:i % 2 + 1].copy_(lt, non_blocking=True)
            loss_ev[i % 2].record()
            if i > 0:
                loss_ev[(i - 1) % 2].synchronize()
                losses.append(float(loss_h[(i - 1) % 2]))
            _, nb = delta_tick(i, device_only=False)
            d2h += nb + 8
        if pend[0] is not None:  # the last tick's payloads, inside the timed region
            d2h += sum(len(p) for p in pend[0].result(copy=False))
            pend[0] = None
        loss_ev[(args.steps - 1) % 2].synchronize()
        losses.append(float(loss_h[(args.steps - 1) % 2]))
        assert len(losses) == args.steps and all(np.isfinite(losses))
        e1.record()
        torch.cuda.synchronize()
        gc.enable()
        ems = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
        if pg is not None:
            dist.all_reduce(ems, op=dist.ReduceOp.MAX)
        e2e = {"value": args.views * args.steps / (float(ems.item()) / 1e3), "unit": "views/s",
               "h2d_bytes_per_step": h2d * world, "d2h_bytes_per_step": d2h // args.steps,
               "path": "optim.step (ground truth H2D from pinned host memory, loss read back) + the tick's "
                       "TENSOR_DELTA frames (device CRC-32) read back into pinned host memory"}


    # per-class device time, launch count and the dominant kernel's launch
    # time: the same steps again (after the e2e record) (library CUDA events around every launch
    # group), the view lanes serialised on one stream so each kernel is
    # timed alone rather than stretched by a concurrent lane
    lanes = optim_mod.VIEW_LANES
    optim_mod.VIEW_LANES = 1
    _lib.set_timing(c, True)
    _lib.get_timing(c, reset=True)
    for i in range(args.steps):
        one_step(args.warmup + args.steps + i)
    torch.cuda.synchronize()
    kt, counters = _lib.get_timing(c, reset=True)
    _lib.set_timing(c, False)
    optim_mod.VIEW_LANES = lanes

    # ---- the backward's throughput mode (float atomics, ss_render_opts.deterministic = 0),
    # same workload and timing; the headline `value` is the deterministic mode
    atomics = None
    if not args.step_only or args.atomics:
        atomics = atomics_bench(args, dm, state, views, ws, pg, dev, delta_tick, torch)

    # ---- delta encoder alone (rank 0): per-frame set, raw, device-resident
    enc = None
    extras = rank == 0 and not args.step_only
    if extras:
        enc = encoder_bench(c, _lib, args, torch)
        enc["snapshot"] = snapshot_bench(dm, torch)

    # ---- BASELINE configs 2 and 4 (rank 0, after the timed runs)
    config2 = config4 = None
    if extras:
        config2 = config2_bench(args, dev, torch)
        config4 = {f"sh{d}": config4_bench(args, dev, torch, degree=d) for d in (1, 3)}

    # ---- pool maintenance of this model, rank 0
    pool_rec = zlib_rec = engine_rec = None
    if extras:
        pool_rec = pool_bench(dm, solo_state(), poses, intr, torch)
        zlib_rec = zlib_tick_bench(dm, base_m, base_l, torch)

    # ---- config 5: client-viewpoint rendering, views sharded over the ranks (no collective)
    client_rec = None
    if not args.no_e2e and not args.step_only:
        client_rec = client_render_bench(args, rank, world, pg, dev, torch)

    # ---- the engine stand-in and a full server tick on the device (§8f rank 4), rank 0,
    # after the timed runs (it trains the model further and holds its own buffers)
    if extras:
        engine_rec = engine_bench(poses, intr, torch)
        engine_rec["live_tick"] = live_tick_bench(dm, solo_state(), poses, intr, light, torch)

    if rank != 0:
        if pg is not None:
            dist.destroy_process_group()
        return

    per_step = {k: v[0] / args.steps for k, v in kt.items()}
    evals_per_view = counters[0] / max(1, args.steps * len(mine))
    launches = int(counters[1])
    dom = max(per_step, key=per_step.get)
    roof = roofline(dom, per_step, kt, counters, args, len(mine), fp32_peak)
    roof["hbm_alternative"] = step_hbm_roofline(args, dm, int(ws.bins_status[1].item()), ms_per_step, len(mine))

    cpu = None
    if not args.no_cpu_baseline:
        cpu = cpu_baseline(model_h, tgt_h, poses, intr, light)
        if not args.step_only:
            cpu["encoders"] = cpu_encoder_baseline(args)

    out = {"metric": METRIC, "value": value, "unit": "views/s", "n_gpus": world, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "f32", "data": "synthetic",
           "config": workload_config(args), "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
           "gpu_launches": launches, "clocks": clock_rec,
           "kernel_ms_per_step": {k: round(v, 4) for k, v in per_step.items()},
           "atomics_mode": atomics, "config2": config2, "config4": config4,
           "evaluated_pairs_per_view": evals_per_view,
           "delta_encode": enc, "pool_maintenance": pool_rec, "server_tick_zlib": zlib_rec, "engine": engine_rec, "client_render": client_rec, "fp32_peak_tflops_measured": fp32_peak,
           "precision": "fp64 preprocess/windows/depth keys, fp32 blend + chain rule, fp64 Adam moments"}
    print(json.dumps(out), flush=True)
    if pg is not None:
        dist.destroy_process_group()


def config2_bench(args, dev, torch, n=500_000, n_views=4, ticks=30):
    """BASELINE config 2: 500k Gaussians, SH degree 3, 4 views of
    1920x1080 per step, single GPU, each server tick = one optimizer step +
    the deltas due per DEFAULT_DELTA_PERIODS (ref server.py:57-64; raw,
    compression_id 0), the baselines reset from the decoded snapshot first.
    30 ticks cover every period.  Device time with CUDA events."""
    from paper_2604_02851_b200 import _lib, synth
    from paper_2604_02851_b200.model import DeviceModel
    from paper_2604_02851_b200.optim import OptimizerState, ReferenceView, StepWorkspace, step
    from paper_2604_02851_b200.protocol import DeltaTicker, PayloadBuffer, encode_snapshot_device
    from paper_2604_02851_b200.render import render_device
    host = synth.random_field(n, 3, args.width, args.height, seed=5)
    dm = DeviceModel.from_host(host, dev.index)
    tgt = DeviceModel.from_host(synth.target_model(host, seed=6), dev.index)
    poses = synth.ring_poses(n_views)
    intr = synth.intrinsics(args.width, args.height)
    light = synth.light()
    bg = np.array([0.05, 0.05, 0.08])
    views = [ReferenceView(p, intr, render_device(tgt, p, intr, light, background=bg), light, bg) for p in poses]
    del tgt
    lo, hi = host.means.min(0), host.means.max(0)
    state = OptimizerState(dm, scene_extent=float(np.linalg.norm(hi - lo) / 2))
    ws = StepWorkspace(dm)
    bm = torch.empty((dm.count, 3), dtype=torch.float32, device=dev)
    bl = torch.empty((dm.count, 3), dtype=torch.float32, device=dev)
    encode_snapshot_device(dm, 0, None, bm, bl)
    a = dm.active_count
    ticker = DeltaTicker(dm, {0: bm[:a], 1: bl[:a]}, {k: PayloadBuffer(1 << 20, dev) for k in range(7)})

    def tick(i):
        step(dm, state, views, workspace=ws, sync_loss=False)
        due = [attr for attr in DELTA_ORDER if i % DELTA_PERIODS[attr] == 0]
        ticker(due)
        return a * len(due)

    for i in range(3):
        tick(i)
    ws.flush()
    torch.cuda.synchronize()
    c = _lib.ctx(dev.index)
    _lib.set_timing(c, True)
    _lib.get_timing(c, reset=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rows = sum(tick(i) for i in range(ticks))
    e1.record()
    torch.cuda.synchronize()
    kt, _ = _lib.get_timing(c, reset=True)
    _lib.set_timing(c, False)
    ws.flush()
    ms = e0.elapsed_time(e1)
    enc_ms = kt["encoders"][0]
    return {"workload": f"config2: {n} Gaussians SH3, {n_views} views {args.width}x{args.height} per step, 1 GPU, "
                        "one step + the due deltas per tick (DEFAULT_DELTA_PERIODS, raw)",
            "views_per_s": n_views * ticks / (ms / 1e3), "tick_ms": ms / ticks, "ticks": ticks,
            "delta_rows_per_tick": rows / ticks, "encoder_ms_per_tick": enc_ms / ticks,
            "encoder_gaussians_per_s": rows / (enc_ms / 1e3) if enc_ms > 0 else None,
            "note": "device time (CUDA events) over the ticks; encoder = the batched delta launch's own time"}


def config4_bench(args, dev, torch, n=2_000_000, degree=1, ticks=60):
    """BASELINE config 4: a 60 Hz dynamic tick over a 2M-row
    model (SH degree 1 as config_dynamics, and a degree-3 variant), 20 % of
    the rows on 3 rigid objects moving at t = tick/60 (rotation + bounce /
    oscillation), the light yawing at 60 deg/s, optimizer off.  Per tick, all
    on the device: the rigid transforms (ref model.py:389-404), the light
    camera's 1024x1024 ortho depth of the engine scene (ref engine.py:200-219),
    light visibility with the device change flag (ref render.py:350-368,
    server.py:406-409) and, when it flipped, the LightVisibility packet, then
    every due delta (ref server.py:488-493; raw, compression_id 0).  The
    moved rows exceed the gate and go out as sparse means residuals
    (SURVEY §8d).  Reported: the device time per tick against the 16.7 ms
    budget, the wall clock per tick including the host read of the change
    flag and of the tick's payloads (pinned), and rows encoded per second."""
    import math as _m
    from paper_2604_02851_b200 import engine, synth
    from paper_2604_02851_b200.model import DeviceModel
    from paper_2604_02851_b200.objects import ObjectRegistry
    from paper_2604_02851_b200.protocol import DeltaTicker, PayloadBuffer, encode_light_visibility_device
    from paper_2604_02851_b200.render import update_light_visibility
    from paper_2604_02851_b200.scene import scene_from_dict
    host = synth.random_field(n, degree, args.width, args.height, seed=9, object_fraction=0.2)
    dm = DeviceModel.from_host(host, dev.index)
    reg = ObjectRegistry(dev.index)
    for oid in (1, 2, 3):
        reg.set_transform(oid, np.array([1.0, 0.0, 0.0, 0.0]), np.zeros(3))
    reg.refresh_locals(dm)
    scene = scene_from_dict(ENGINE_SCENE)
    lo, hi = host.means.min(0) - 0.25, host.means.max(0) + 0.25
    a = dm.active_count
    base_m, base_l = dm.means.clone(), dm.log_scales.clone()
    ticker = DeltaTicker(dm, {0: base_m[:a], 1: base_l[:a]}, {k: PayloadBuffer(1 << 20, dev) for k in range(7)})
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    vis_out = PayloadBuffer(4 + (n + 7) // 8, dev)
    pinned = torch.empty(256 << 20, dtype=torch.uint8).pin_memory()

    def transforms(t):
        out = {}
        for k, oid in enumerate((1, 2, 3)):
            ang = (0.5 + 0.3 * k) * t
            ax = np.array([0.0, 1.0, 0.2 * k])
            ax = ax / np.linalg.norm(ax)
            q = np.concatenate([[_m.cos(ang / 2)], _m.sin(ang / 2) * ax])
            tr = np.array([0.3 * _m.sin(2.0 * t + k), abs(_m.sin(3.0 * t + k)) * 0.2, 0.1 * _m.cos(t + k)])
            out[oid] = (q, tr)
        return out

    def tick(i, read):
        t = i / 60.0
        for oid, (q, tr) in transforms(t).items():
            reg.apply_transform(dm, oid, q, tr, return_rows=False)
        yaw = _m.radians(60.0) * t
        d = np.array([0.3 * _m.cos(yaw) - 0.2 * _m.sin(yaw), -1.0, 0.3 * _m.sin(yaw) + 0.2 * _m.cos(yaw)])
        lcam = engine.build_light_camera(lo, hi, d / np.linalg.norm(d), 1024)
        depth = engine.render_ortho_depth(scene, lcam, as_tensor=True)
        flag.zero_()
        update_light_visibility(dm, depth, lcam, changed=flag)
        encode_light_visibility_device(dm.light_visibility, vis_out)
        due = [attr for attr in DELTA_ORDER if i % DELTA_PERIODS[attr] == 0 and not (attr == 5 and degree == 0)]
        ticker(due)
        nbytes = 0
        if read:  # the server's host side: the change flag, then the frames' bytes
            sent_vis = bool(flag.item())
            lens = [int(ticker.outs[k].length.item()) for k in due]
            off = 0
            for k, ln in zip(due, lens):
                pinned[off:off + ln].copy_(ticker.outs[k].data[:ln], non_blocking=True)
                off += ln
            if sent_vis:
                ln = int(vis_out.length.item())
                pinned[off:off + ln].copy_(vis_out.data[:ln], non_blocking=True)
                off += ln
            torch.cuda.current_stream().synchronize()
            nbytes = off
        return a * len(due), nbytes

    for i in range(3):
        tick(i, True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rows = sum(tick(3 + i, False)[0] for i in range(ticks))
    e1.record()
    torch.cuda.synchronize()
    dev_ms = e0.elapsed_time(e1) / ticks
    wall, nb = [], 0
    for i in range(ticks):
        w0 = time.perf_counter()
        _, b = tick(3 + ticks + i, True)
        wall.append((time.perf_counter() - w0) * 1e3)
        nb += b
    return {"workload": f"config4: {n} rows SH{degree}, 20 % on 3 rigid objects, light yaw 60 deg/s, 1024^2 light "
                        "depth, 60 Hz tick (transforms + light visibility + packet + due deltas, raw), optimizer off",
            "tick_ms_device": dev_ms, "tick_ms_wall_p50": float(np.median(wall)), "tick_ms_wall_max": float(max(wall)),
            "budget_ms": 1000.0 / 60.0, "within_budget": float(np.median(wall)) <= 1000.0 / 60.0,
            "rows_encoded_per_s": rows / (dev_ms * ticks / 1e3), "bytes_per_tick": nb / ticks,
            "note": "device time per tick (CUDA events, no host reads) and wall clock per tick with the host "
                    "reading the change flag and the payload bytes into pinned memory"}


def atomics_bench(args, dm, state, views, ws, pg, dev, delta_tick, torch, steps=None):
    """The timed loop again with the backward's throughput mode: each (tile,
    splat) pair's sums go into the splat's record with float atomics (no
    per-pair partials, no fixed-order partial sum).  Same step otherwise;
    device time with CUDA events, max over ranks."""
    import torch.distributed as dist
    from paper_2604_02851_b200.optim import step
    k = steps or args.steps
    for i in range(2):
        step(dm, state, views, workspace=ws, sync_loss=False, deterministic=False)
    torch.cuda.synchronize()
    if pg is not None:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(k):
        step(dm, state, views, workspace=ws, sync_loss=False, deterministic=False)
        delta_tick(i)
    e1.record()
    torch.cuda.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if pg is not None:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())
    return {"value": args.views * k / (ms / 1e3), "unit": "views/s", "ms_per_step": ms / k, "steps": k,
            "note": "optim.step(deterministic=False): per-(tile, splat) sums added with float atomics into the "
                    "per-row screen-space records (no partials, no fixed-order sum); the headline value is the "
                    "deterministic mode"}


def ctypes_peak(c):
    import ctypes
    v = ctypes.c_double(0)
    c.check(c.lib.ss_measure_fp32_peak(c.handle, ctypes.byref(v)))
    return v.value


def encoder_bench(c, _lib, args, torch, reps=20):
    """Delta-encode Gaussians/s on config 4's model size (2M rows, SH degree 1
    as in config_dynamics): the per-frame set (means, log_scales, opacity, DC;
    raw) in one batched call per tick.  Baselines are offset so both residual
    attributes take the dense path (the common case while rows are being
    optimised) and re-armed before every tick."""
    from paper_2604_02851_b200 import synth
    from paper_2604_02851_b200.model import DeviceModel
    from paper_2604_02851_b200.protocol import DeltaTicker, PayloadBuffer
    n = 2 * args.n
    dm = DeviceModel.from_host(synth.random_field(n, 1, args.width, args.height, seed=3), c.device)
    a = dm.active_count
    per_frame = (0, 1, 3, 4)
    ref_m = (dm.means - 2e-3).contiguous()
    ref_l = (dm.log_scales - 2e-3).contiguous()
    bm, bl = ref_m.clone(), ref_l.clone()
    bufs = {k: PayloadBuffer(1 << 20, dm.device) for k in range(7)}
    tick = DeltaTicker(dm, {0: bm, 1: bl}, bufs)
    for _ in range(3):
        tick(per_frame)
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    _lib.set_timing(c, True)
    _lib.get_timing(c, reset=True)
    # between ticks: re-arm the baselines, then stream a 256 MB buffer through
    # L2 so the re-arm's dirty lines are written back outside the timed
    # region (in the server loop the optimizer step sits between two ticks)
    # and every tick starts with the inputs in DRAM
    flush, clean = l2_flush_buffers(dm.device, torch)
    for e0, e1 in ev:
        bm.copy_(ref_m)
        bl.copy_(ref_l)
        l2_flush(flush, clean)
        e0.record()
        tick(per_frame)
        e1.record()
    torch.cuda.synchronize()
    kt, _ = _lib.get_timing(c, reset=True)
    _lib.set_timing(c, False)
    ms = sum(e0.elapsed_time(e1) for e0, e1 in ev) / reps
    dev_ms = kt["encoders"][0] / max(1, kt["encoders"][1])
    # algorithmic bytes per row: dense residual = 4d cur + 4d base read + 4d base write
    # + code bytes; absolute = 4d read + code bytes
    bytes_per_row = (12 + 12 + 12 + 6) + (12 + 12 + 12 + 3) + (4 + 1) + (12 + 3)
    gbs = bytes_per_row * a / (dev_ms * 1e-3) / 1e9
    peak = measured_peaks().get("hbm_gbs", 6551.4)
    payload = sum(int(bufs[k].length.item()) for k in per_frame)
    out = {"value": a / (ms * 1e-3), "unit": "Gaussians/s", "rows": a, "sh_degree": 1, "ms_per_tick": ms,
           "kernel_ms_per_tick": dev_ms, "payload_bytes_per_tick": payload,
           "set": "means+log_scales (dense residual, baseline advanced) + opacity + DC, raw, one batched call",
           "l2": "flushed between ticks (after the baseline re-arm: 256 MB written, then 256 MB read; bench.l2_flush)",
           "roofline": {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s", "frac": gbs / peak,
                        "traffic": committed_traffic("delta_encode"), "traffic_unit": "bytes/tick (ncu, profiles/)",
                        "algorithmic_bytes_per_tick": bytes_per_row * a, "bytes_per_row": bytes_per_row,
                        "note": "achieved = algorithmic bytes / kernel time of the tick's launch"}}
    out["client_apply"] = ingest_bench(dm, tick, per_frame, ref_m, ref_l, bm, bl, torch)
    del dm
    return out


def l2_flush_buffers(device, torch):
    return (torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=device),
            torch.zeros(64 * 1024 * 1024, dtype=torch.float32, device=device))


def l2_flush(flush, clean):
    """L2 flush before a timed encoder call: write 256 MB (every line of the
    126 MB L2 replaced, earlier dirty data written back), then read another
    256 MB, so the timed call starts with its inputs in DRAM and no dirty
    lines of the flush itself left to write back inside its region (ncu's
    own cache control flushes and invalidates the same way)."""
    flush.add_(1.0)
    clean.sum()


def snapshot_bench(dm, torch, reps=10):
    """K11 on the bench model (1M rows, SH degree 3): the profile-0 snapshot
    (raw, compression 0) plus the server's baseline reset outputs, device time
    per encode with L2 flushed before each; roofline on the algorithmic bytes
    of DESIGN.md K11 (244 B read + 38 B written per row at degree 3)."""
    from paper_2604_02851_b200.protocol import PayloadBuffer, encode_snapshot_device
    out = PayloadBuffer(1 << 20, dm.device)
    bm = torch.empty_like(dm.means)
    bl = torch.empty_like(dm.log_scales)
    for _ in range(2):
        encode_snapshot_device(dm, 0, out, bm, bl)
    flush, clean = l2_flush_buffers(dm.device, torch)
    ts = []
    for _ in range(reps):
        l2_flush(flush, clean)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        encode_snapshot_device(dm, 0, out, bm, bl)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts))
    rows = dm.count
    alg = rows * (244 + 38)
    peak = measured_peaks().get("hbm_gbs", 6551.4)
    gbs = alg / (ms * 1e-3) / 1e9
    return {"value": rows / (ms * 1e-3), "unit": "Gaussians/s", "rows": rows, "sh_degree": dm.sh_degree,
            "ms_per_snapshot": ms, "payload_bytes": int(out.length.item()),
            "roofline": {"bound": "hbm", "achieved": gbs, "peak": peak, "unit": "GB/s", "frac": gbs / peak,
                         "algorithmic_bytes": alg},
            "note": "device time per encode (profile 0, raw) incl. the decoded means/log-scales for the baseline "
                    "reset; L2 flushed before each (256 MB written, then 256 MB read; bench.l2_flush)"}


def ingest_bench(dm, tick, per_frame, ref_m, ref_l, bm, bl, torch, reps=10):
    """Client side of the same tick: the payloads applied
    to a device replica through protocol.apply_delta (host bytes in, parse +
    H2D + device validate + apply), rows/s over the per-frame set."""
    from paper_2604_02851_b200.protocol import DeviceBaselines, apply_delta
    bm.copy_(ref_m)
    bl.copy_(ref_l)
    tick(per_frame)
    payloads = tick.read(per_frame)
    rep_model = dm.clone()
    base = DeviceBaselines(ref_m.clone(), ref_l.clone(), 0)
    for p in payloads:  # warm-up
        apply_delta(rep_model, base, p, 0, 0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        base.means.copy_(ref_m)
        base.log_scales.copy_(ref_l)
        for p in payloads:
            apply_delta(rep_model, base, p, 0, 0)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3 / reps
    same = bool(torch.equal(rep_model.means[:dm.active_count], bm[:dm.active_count]))
    return {"value": dm.active_count / (ms * 1e-3), "unit": "Gaussians/s", "ms_per_tick": ms,
            "payload_bytes_per_tick": sum(len(p) for p in payloads),
            "replica_equals_server_baseline": same,
            "note": "wall clock per tick of 4 apply_delta calls (host payload bytes -> device replica), incl. baseline re-arm copies"}


def zlib_tick_bench(dm, base_m, base_l, torch, reps=3):
    """The reference server's default stream (compression_id 1) for tick 0
    (all six attributes) of the 1M-row model: DeltaEmitter with the blocks
    deflated serially vs on parallel host threads."""
    from paper_2604_02851_b200 import protocol as P
    base = P.DeviceBaselines(base_m.clone(), base_l.clone(), 0)
    em = P.DeltaEmitter(dm, base, compression_id=1)
    em.tick(0)
    ref_m, ref_l = base.means.clone(), base.log_scales.clone()
    a = dm.active_count
    raws = None
    t_par = t_ser = 0.0
    for _ in range(reps):
        base.means.copy_(ref_m)
        base.log_scales.copy_(ref_l)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        out = em.tick(0)
        t_par += time.perf_counter() - t0
    em_raw = P.DeltaEmitter(dm, base, compression_id=0)
    base.means.copy_(ref_m)
    base.log_scales.copy_(ref_l)
    raws = [p for _, p in em_raw.tick(0)]
    for _ in range(reps):
        t0 = time.perf_counter()
        ser = [P._recompress_delta(r, 1) for r in raws]
        t_ser += time.perf_counter() - t0
    assert ser == [p for _, p in out]
    # frame envelope CRC of the raw stream's payloads: device (ss_crc32) vs host zlib.crc32
    import zlib
    base.means.copy_(ref_m)
    base.log_scales.copy_(ref_l)
    bufs = [em_raw._outs[int(at)] for at, _ in em_raw.tick(0)]  # the same payloads as `raws`, still in HBM
    for b in bufs:
        P.crc32_device(b.data, b.length)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    dev_crc = [P.crc32_device(b.data, b.length) for b in bufs]
    e1.record()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    host_crc = [zlib.crc32(r) for r in raws]
    t_crc = time.perf_counter() - t0
    assert [int(c.item()) & 0xFFFFFFFF for c in dev_crc] == host_crc
    return {"rows": a, "attributes": len(out), "raw_bytes": sum(len(r) for r in raws),
            "frame_crc_us_device": e0.elapsed_time(e1) * 1e3, "frame_crc_ms_host_zlib": t_crc * 1e3,
            "zlib_bytes": sum(len(p) for _, p in out), "tick_ms_parallel_zlib": t_par * 1e3 / reps,
            "zlib_stage_ms_serial": t_ser * 1e3 / reps,
            "note": "tick = device encode + readback + per-attribute deflate on host threads (byte-identical)"}


ENGINE_SCENE = {  # the engine stand-in's test scene (tests/golden/make_golden.py ENGINE_SCENES)
    "background": [0.05, 0.05, 0.08],
    "light": {"direction": [-0.4, -1.0, 0.3], "intensity": [0.8, 0.8, 0.8], "ambient": [0.2, 0.2, 0.2]},
    "objects": [
        {"id": 0, "shape": {"kind": "plane", "point": [0, 0, 0], "normal": [0, 1, 0], "extent": [4.0, 4.0]},
         "albedo": {"kind": "checker", "colors": [[0.9, 0.9, 0.9], [0.2, 0.25, 0.35]], "scale": 1.0}},
        {"id": 1, "shape": {"kind": "sphere", "center": [0, 0.5, 0], "radius": 0.5},
         "albedo": {"kind": "solid", "color": [0.8, 0.2, 0.15]}},
        {"id": 2, "shape": {"kind": "box", "center": [1.2, 0.4, -0.6], "half_extents": [0.3, 0.4, 0.25]},
         "albedo": {"kind": "checker", "colors": [[0.1, 0.7, 0.2], [0.9, 0.8, 0.1]], "scale": 0.25}},
    ]}


def client_render_bench(args, rank, world, pg, dev, torch, n=2_000_000, views=64, reps=2):
    """Config 5: 64 client viewpoints of a 2M-Gaussian SH3 model at 1080p,
    the viewpoints sharded round-robin over the ranks with no collective
    (SURVEY §8e); frames/s of the whole job, timed on the device (max over
    ranks).  The model is the synthetic field, replicated per rank."""
    import torch.distributed as dist
    from paper_2604_02851_b200 import synth
    from paper_2604_02851_b200.model import DeviceModel
    from paper_2604_02851_b200.render import render_device_many
    m = DeviceModel.from_host(synth.random_field(n, 3, args.width, args.height, seed=7), dev.index)
    intr = synth.intrinsics(args.width, args.height)
    light = synth.light()
    allp = synth.ring_poses(views, radius=0.6)
    mine = allp[rank::world]
    lanes = 4
    outs = [torch.empty((args.height, args.width, 3), dtype=torch.float32, device=dev) for _ in range(lanes)]
    render_device_many(m, mine[:lanes], intr, light, outs=outs, lanes=lanes)
    torch.cuda.synchronize()
    if pg is not None:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        render_device_many(m, mine, intr, light, outs=outs, lanes=lanes)
    e1.record()
    torch.cuda.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if pg is not None:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())
    del m
    return {"value": views * reps / (ms / 1e3), "unit": "frames/s", "viewpoints": views, "gaussians": n,
            "sh_degree": 3, "resolution": [args.width, args.height], "ms_per_frame_per_gpu": ms / (reps * len(mine)),
            "note": "render_device_many (per viewpoint: preprocess, depth sort, binning, tile sort, forward; 4 "
                    "lanes of streams); viewpoints sharded round-robin over the ranks, no collective; device time, "
                    "max over ranks"}


def engine_bench(poses, intr, torch, reps=5):
    """SURVEY §8f rank 4 on the device: the ray-cast ground truth of the
    step's 8 views at 1080p (float32, left in HBM for the optimiser), and one
    expansion round (8 dome cameras at 256x256: capture buffers, cull, init)."""
    from paper_2604_02851_b200 import engine
    from paper_2604_02851_b200.geometry import look_at
    from paper_2604_02851_b200.scene import scene_from_dict
    scene = scene_from_dict(ENGINE_SCENE)
    views = [look_at(np.array([3.0 * np.cos(a), 2.2, 3.0 * np.sin(a)]), np.array([0.0, 0.3, 0.0]))
             for a in np.linspace(0, 2 * np.pi, len(poses), endpoint=False)]
    outs = [engine.render_ground_truth_device(scene, p, intr) for p in views]
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        for p, o in zip(views, outs):
            engine.render_ground_truth_device(scene, p, intr, out=o)
    e1.record()
    torch.cuda.synchronize()
    gt_ms = e0.elapsed_time(e1) / (reps * len(views))
    rig, rintr = engine.build_dome_rig(np.array([0.0, 0.3, 0.0]), 0.4, 8, 3.0, width=256, height=256, fov_y=1.3)
    t = []
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        bufs = [engine.capture_input_buffers(scene, p, rintr, as_tensors=True) for p in rig]
        sb = engine.cull_input_samples(bufs, as_tensors=True)
        batch = engine.init_gaussians(sb, sh_degree=3, as_device=True)
        torch.cuda.synchronize()
        t.append(time.perf_counter() - t0)
    return {"gt_ms_per_view": gt_ms, "gt_megapixels_per_s": intr.width * intr.height / (gt_ms * 1e3),
            "resolution": [intr.width, intr.height], "objects": len(scene.objects),
            "expansion_round_ms": min(t) * 1e3, "expansion_cameras": len(rig), "expansion_samples": sb.count,
            "new_gaussians": batch.count,
            "note": "device time per 1080p ground-truth view (primary + shadow ray per pixel, float64); expansion = "
                    "wall clock of capture_input_buffers x8 + cull_input_samples + init_gaussians"}


def live_tick_bench(dm, state, poses, intr, light_state, torch, ticks=6):
    """One server tick (ref server.py:364-493) with every stage on the device,
    through the public APIs: (3) light-camera ortho depth + light visibility,
    (4) expansion inputs (4 input cameras at 256x256: capture buffers, cull,
    init -- the grid-gated append policy itself is host logic, not timed),
    (5) ray-cast ground truth of the step's views straight into HBM, precull,
    optimize step, grid rebuild, (6) freeze policy, (8) the due deltas as
    TENSOR_DELTA frames read back to pinned host memory.  The engine scene is
    the stand-in test scene (the model is the synthetic 1M field, so the
    images do not depict it: the stage costs are what is measured)."""
    from paper_2604_02851_b200 import engine, pool
    from paper_2604_02851_b200.optim import ReferenceView, StepWorkspace, step
    from paper_2604_02851_b200.protocol import DELTA_ORDER, DeltaTicker, PayloadBuffer
    from paper_2604_02851_b200.render import update_light_visibility
    from paper_2604_02851_b200.scene import scene_from_dict
    scene = scene_from_dict(ENGINE_SCENE)
    gts = [torch.empty((intr.height, intr.width, 3), dtype=torch.float32, device=dm.device) for _ in poses]
    views = [ReferenceView(p, intr, g, light_state, np.zeros(3)) for p, g in zip(poses, gts)]
    lcam = engine.build_light_camera(np.array([-5.0, -1.0, -1.0]), np.array([5.0, 3.0, 9.0]), light_state.direction, 256)
    rig, rintr = engine.build_dome_rig(np.array([0.0, 0.3, 0.0]), 0.4, 4, 3.0, width=256, height=256, fov_y=1.3)
    grid = pool.GridIndex(cell_size=0.5, origin=(0.0, 0.0, 0.0))
    base = {0: dm.means.clone(), 1: dm.log_scales.clone()}
    ticker = DeltaTicker(dm, base, {k: PayloadBuffer(1 << 20, dm.device) for k in range(7)})
    ws = StepWorkspace(dm)
    periods = {0: 1, 1: 1, 2: 10, 3: 1, 4: 1, 5: 30}
    pend = None
    times, stages = [], {}

    def tick(i, record):
        nonlocal pend
        marks = [time.perf_counter()]
        ld = engine.render_ortho_depth(scene, lcam, as_tensor=True)
        update_light_visibility(dm, ld, lcam)
        marks.append(time.perf_counter())
        bufs = [engine.capture_input_buffers(scene, p, rintr, as_tensors=True) for p in rig]
        batch = engine.init_gaussians(engine.cull_input_samples(bufs, as_tensors=True), sh_degree=dm.sh_degree,
                                      as_device=True)
        marks.append(time.perf_counter())
        for p, g in zip(poses, gts):
            engine.render_ground_truth_device(scene, p, intr, out=g)
        subset = pool.precull(dm, grid, poses, intr, as_tensor=True) if grid.cells is not None else None
        step(dm, state, views, index_subset=subset, workspace=ws, sync_loss=False)
        grid.rebuild(dm)
        pool.freeze_policy(dm, state, age_threshold=120, grad_threshold=3e-4)
        marks.append(time.perf_counter())
        due = [int(a) for a in DELTA_ORDER if i % periods[int(a)] == 0]
        ticker(due)
        done, pend = pend, ticker.read_async(due, frame_epoch=1)
        nbytes = sum(len(f) for f in done.result(copy=False)) if done is not None else 0
        marks.append(time.perf_counter())
        if record:
            for k, (a, b) in zip(("light", "expansion_inputs", "ground_truth+optimize+pool", "delta_frames"),
                                 zip(marks, marks[1:])):
                stages.setdefault(k, []).append((b - a) * 1e3)
        return batch.count, nbytes

    for i in range(2):
        tick(i, False)
    torch.cuda.synchronize()
    for i in range(ticks):
        t0 = time.perf_counter()
        new_rows, nbytes = tick(i, True)
        times.append(time.perf_counter() - t0)
    pend.result(copy=False)
    torch.cuda.synchronize()
    ms = float(np.median(times)) * 1e3
    return {"tick_ms": ms, "ticks_per_s": 1e3 / ms, "views": len(poses), "resolution": [intr.width, intr.height],
            "gaussians": dm.active_count, "new_gaussians_per_tick": new_rows, "frame_bytes_read": nbytes,
            "stage_ms_host_wall": {k: float(np.median(v)) for k, v in stages.items()},
            "note": "wall clock per tick (median of %d), host enqueue included; stages are host wall clock per "
                    "stage (asynchronous GPU work can land in a later stage)" % ticks}


def pool_bench(dm, state, poses, intr, torch, reps=5):
    """Per-tick pool maintenance on the 1M-row model:
    GridIndex.rebuild, precull against the step's 8 cameras and
    freeze_policy, each as the reference API call (host result)."""
    from paper_2604_02851_b200 import pool
    from paper_2604_02851_b200.geometry import CameraIntrinsics
    g = pool.GridIndex(cell_size=0.5, origin=(0.0, 0.0, 0.0))
    ci = CameraIntrinsics(width=intr.width, height=intr.height, fov_y=intr.fov_y, near=intr.near, far=100.0)

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            out = fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) * 1e3 / reps, out

    t_grid, _ = timed(lambda: g.rebuild(dm))
    t_pre, kept = timed(lambda: pool.precull(dm, g, poses, ci))
    t_frz, frz = timed(lambda: pool.freeze_policy(dm, state, 100, 1e-4))
    return {"rows": dm.count, "cells": int(g.cell_lens.shape[0]), "grid_rebuild_ms": t_grid, "precull_ms": t_pre,
            "precull_rows": int(kept.size), "freeze_policy_ms": t_frz,
            "note": "wall clock per call incl. the host readback of the result (reference: ~1.08 s per 1M-row rebuild on CPU, SURVEY §8f)"}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            return json.load(f)
    return {}


def _committed(key):
    p = os.path.join(ROOT, "profiles", "r02_traffic.json")
    try:
        with open(p) as f:
            return json.load(f).get(key, {})
    except (OSError, ValueError):
        return {}


def committed_traffic(key):
    """DRAM bytes per launch of a kernel class from this round's committed ncu
    capture (profiles/r01_traffic.json); None when absent."""
    e = _committed(key)
    return e.get("bytes_per_launch", e.get("bytes_per_tick"))


def step_hbm_roofline(args, dm, pairs_per_view, ms_per_step, local_views):
    """SURVEY §8d optimize roofline (i), the HBM view of the whole step:
    per view N (2P + 64) + pairs x 24 + H W (12 GT + 12 image + 4 T) + a P
    bytes, plus Adam's 7 a P per step (P = 4 (11 + 3B) bytes per row), over
    the measured step time.  Reported beside the FP32 roofline of the
    dominant kernel (SURVEY: take the larger fraction -- the FP32 one)."""
    peaks = measured_peaks()
    hbm = peaks.get("hbm_gbs", 6551.4)
    B = (dm.sh_degree + 1) ** 2
    P = 4 * (11 + 3 * B)
    n, a = dm.count, dm.active_count
    px = args.width * args.height
    per_view = n * (2 * P + 64) + pairs_per_view * 24 + px * 28 + a * P
    per_step = local_views * per_view + 7 * a * P
    gbs = per_step / (ms_per_step * 1e-3) / 1e9
    return {"bound": "hbm", "achieved": gbs, "peak": hbm, "unit": "GB/s", "frac": gbs / hbm,
            "bytes_per_step": per_step, "pairs_per_view": pairs_per_view,
            "note": "whole-step algorithmic bytes (SURVEY §8d (i)) over the step time; pairs = the largest "
                    "per-view (tile, splat) count of the run"}


def roofline(dom, per_step, kt, counters, args, local_views, fp32_peak):
    """Roofline of the dominant kernel class (per launch = per view)."""
    peaks = measured_peaks()
    hbm = peaks.get("hbm_gbs", 6551.4)
    ms_launch = kt[dom][0] / max(1, kt[dom][1])
    evals = counters[0] / max(1, kt["blend_forward"][1])  # T-gated pairs per forward launch
    px = args.width * args.height
    # algorithmic FP32 work per T-gated pair (SURVEY §8d convention): 22 fwd, 60 bwd
    flops = {"blend_forward": 22 * evals, "blend_backward": 60 * evals}.get(dom)
    if flops is not None:
        tf = flops / (ms_launch * 1e-3) / 1e12
        return {"bound": "fp32", "kernel": dom, "achieved": tf, "peak": fp32_peak, "unit": "TFLOP/s",
                "frac": tf / fp32_peak, "traffic": committed_traffic(dom), "traffic_unit": "bytes/launch (ncu, profiles/)",
                "ms_per_launch": ms_launch,
                "work_per_launch": f"{evals:.4g} T-gated (pixel, splat) pairs x {22 if dom == 'blend_forward' else 60} FLOP",
                "peak_source": "measured FMA probe (ss_measure_fp32_peak)",
                "hbm_peak_gbs": hbm, "ncu": _committed(dom).get("ncu")}
    return {"bound": "hbm", "kernel": dom, "achieved": None, "peak": hbm, "unit": "GB/s", "frac": None,
            "traffic": None, "ms_per_launch": ms_launch}


def cpu_encoder_baseline(args):
    """The oracle port of the encoders on one host core, full size (SURVEY
    §8d): the per-frame delta set of bench.py's encoder workload (2M rows
    SH1: dense means / log-scale residuals, opacity, DC; raw) and the
    profile-0 snapshot of the 1M-row SH3 model (raw)."""
    from oracle import codec as oc
    from paper_2604_02851_b200 import synth
    m = synth.random_field(2 * args.n, 1, args.width, args.height, seed=3)
    a = m.active_count
    base_m, base_l = m.means - np.float32(2e-3), m.log_scales - np.float32(2e-3)
    t0 = time.perf_counter()
    oc.delta_payload(0, m.means[:a], base_m[:a], None, 0)
    oc.delta_payload(1, m.log_scales[:a], base_l[:a], None, 0)
    oc.delta_payload(3, m.logit_opacities[:a], None, None, 0)
    oc.delta_payload(4, m.sh_coeffs[:a, :, 0], None, None, 0)
    t_delta = time.perf_counter() - t0
    del m
    s = synth.random_field(args.n, 3, args.width, args.height, seed=0)
    t0 = time.perf_counter()
    oc.snapshot_payload(s.means, s.log_scales, s.quaternions, s.logit_opacities, s.sh_coeffs, s.light_visibility,
                        s.object_ids, s.active_count, s.sh_degree, 0, 0)
    t_snap = time.perf_counter() - t0
    return {"delta_per_frame_set": {"value": a / t_delta, "unit": "Gaussians/s", "seconds": t_delta, "rows": a,
                                    "cores": 1, "kind": "port"},
            "snapshot": {"value": args.n / t_snap, "unit": "Gaussians/s", "seconds": t_snap, "rows": args.n,
                         "cores": 1, "kind": "port"},
            "note": "oracle numpy port of encode_delta / encode_snapshot (raw), one host core, full size"}


def cpu_baseline(model, tgt, poses, intr, light_state):
    """Oracle port, 1 process, one view on a centre crop, extrapolated."""
    from oracle import raster as orr
    light, jobs, factor = cpu_sample_setup(model, tgt, poses[:1], intr, light_state)
    ccam, rows, gt = jobs[0]
    t0 = time.perf_counter()
    orr.backward(model, ccam, light, gt, (0.05, 0.05, 0.08), rows, True)
    t = time.perf_counter() - t0
    return {"value": 1.0 / (t * factor), "unit": "views/s", "cores": 1, "kind": "port",
            "sample": (f"oracle numpy float64 backward of 1 view on a centre crop of 1/{factor:.0f} of the "
                       f"1920x1080 frame ({len(rows)} rows meet it), {t:.2f} s, extrapolated x{factor:.0f}")}


def launch_ranks(args) -> int:
    """`bench.py --gpus N` without a torchrun environment: re-run this script
    under torch.distributed.run with N ranks (one per GPU) and return its
    exit code (rank 0 prints the JSON line)."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")  # the communicator lines (NVLS / NVLink paths) go to stderr
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


if __name__ == "__main__":
    a = parse()
    world_env = os.environ.get("WORLD_SIZE")
    if a.impl == "ours" and a.gpus > 1 and world_env is None:
        sys.exit(launch_ranks(a))
    if world_env is not None and a.impl == "ours" and int(world_env) != a.gpus:
        sys.exit(f"--gpus {a.gpus} but WORLD_SIZE={world_env}")
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
