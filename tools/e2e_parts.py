"""The bench's e2e loop with parts toggled: where does e2e lose against value?
    python tools/e2e_parts.py"""
import os, sys, gc
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
from paper_2604_02851_b200.model import DeviceModel
from paper_2604_02851_b200.optim import OptimizerState, ReferenceView, StepWorkspace, step
from paper_2604_02851_b200.protocol import DeltaTicker, PayloadBuffer, encode_snapshot_device, DELTA_ORDER
from paper_2604_02851_b200.render import render_device

sys.argv = sys.argv[:1]
args = bench.parse()
model_h, tgt_h, poses, intr, light = bench.build_workload(args)
dev = torch.device("cuda", 0)
dm = DeviceModel.from_host(model_h, 0)
tgt = DeviceModel.from_host(tgt_h, 0)
bg = np.array([0.05, 0.05, 0.08])
gts = [render_device(tgt, p, intr, light, background=bg) for p in poses]
del tgt
dv = [ReferenceView(p, intr, g, light, bg) for p, g in zip(poses, gts)]
hv = [ReferenceView(p, intr, g.cpu().pin_memory(), light, bg) for p, g in zip(poses, gts)]
lo, hi = model_h.means.min(0), model_h.means.max(0)
state = OptimizerState(dm, scene_extent=float(np.linalg.norm(hi - lo) / 2))
ws = StepWorkspace(dm)
a = dm.active_count
base_m = torch.empty((dm.count, 3), dtype=torch.float32, device=dev)
base_l = torch.empty((dm.count, 3), dtype=torch.float32, device=dev)
encode_snapshot_device(dm, 0, None, base_m, base_l)
ticker = DeltaTicker(dm, {0: base_m[:a], 1: base_l[:a]}, {attr: PayloadBuffer(1 << 20, dev) for attr in DELTA_ORDER})
P = bench.DELTA_PERIODS


def fresh():
    """Every configuration starts from the same model and optimizer state."""
    global dm, state, ws, ticker
    dm = DeviceModel.from_host(model_h, 0)
    state = OptimizerState(dm, scene_extent=float(np.linalg.norm(hi - lo) / 2))
    ws = StepWorkspace(dm)
    encode_snapshot_device(dm, 0, None, base_m, base_l)
    ticker = DeltaTicker(dm, {0: base_m[:a], 1: base_l[:a]}, {attr: PayloadBuffer(1 << 20, dev) for attr in DELTA_ORDER})


def loop(views, tick_mode, loss_mode, steps=20):
    fresh()
    pend = [None]
    loss_h = torch.zeros(2, dtype=torch.float64).pin_memory()
    ev = [torch.cuda.Event(), torch.cuda.Event()]

    def tick(i):
        due = [x for x in DELTA_ORDER if i % P[x] == 0]
        if tick_mode == "none":
            return
        ticker(due)
        if tick_mode == "host":
            p = ticker.read_async(due, frame_epoch=1)
            done, pend[0] = pend[0], p
            if done is not None:
                done.result(copy=False)
    for i in range(3):
        step(dm, state, views, workspace=ws, sync_loss=False)
        tick(i)
    torch.cuda.synchronize()
    gc.collect()
    gc.disable()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(steps):
        lt = step(dm, state, views, workspace=ws, sync_loss=False)
        if loss_mode:
            loss_h[i % 2:i % 2 + 1].copy_(lt, non_blocking=True)
            ev[i % 2].record()
            if i > 0:
                ev[(i - 1) % 2].synchronize()
        tick(i)
    if pend[0] is not None:
        pend[0].result(copy=False)
    e1.record()
    torch.cuda.synchronize()
    gc.enable()
    return e0.elapsed_time(e1) / steps


for name, views, tm, lm in (("device GT, device tick, no loss", dv, "device", False),
                            ("host GT, device tick, no loss", hv, "device", False),
                            ("host GT, no tick, loss", hv, "none", True),
                            ("host GT, device tick, loss", hv, "device", True),
                            ("host GT, host tick, no loss", hv, "host", False),
                            ("host GT, host tick, loss (bench e2e)", hv, "host", True),
                            ("device GT, device tick, no loss", dv, "device", False)):
    print(f"{name:40s} {loop(views, tm, lm):.2f} ms/step", flush=True)
