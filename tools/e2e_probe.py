"""Where does the end-to-end step lose time against the device-resident one?"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2604_02851_b200 import synth
from paper_2604_02851_b200.model import DeviceModel
from paper_2604_02851_b200.optim import OptimizerState, ReferenceView, StepWorkspace, step
from paper_2604_02851_b200.render import render_device

n, V, W, H = 1_000_000, 8, 1920, 1080
model = synth.random_field(n, 3, W, H, seed=0)
tgt = synth.target_model(model, seed=1)
poses, intr, light = synth.ring_poses(V), synth.intrinsics(W, H), synth.light()
dm = DeviceModel.from_host(model, 0)
td = DeviceModel.from_host(tgt, 0)
bg = np.array([0.05, 0.05, 0.08])
gts = [render_device(td, p, intr, light, background=bg) for p in poses]
dv = [ReferenceView(p, intr, g, light, bg) for p, g in zip(poses, gts)]
hv = [ReferenceView(p, intr, g.cpu().pin_memory(), light, bg) for p, g in zip(poses, gts)]
state = OptimizerState(dm, scene_extent=10.0)
ws = StepWorkspace(dm)


def run(views, sync, reps=10):
    for _ in range(2):
        step(dm, state, views, workspace=ws, sync_loss=sync)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(reps):
        step(dm, state, views, workspace=ws, sync_loss=sync)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, (time.perf_counter() - t0) * 1e3 / reps


for name, views, sync in (("device GT, no sync", dv, False), ("device GT, loss sync", dv, True),
                          ("host GT, no sync", hv, False), ("host GT, loss sync", hv, True)):
    print(f"{name:24s} device {run(views, sync)[0]:.2f} ms/step  wall {run(views, sync)[1]:.2f}")
