"""optim.step with index_subset = every row vs None: what does the subset path cost?"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.argv = sys.argv[:1]
import numpy as np
import torch
import bench
from paper_2604_02851_b200 import optim
from paper_2604_02851_b200.model import DeviceModel
from paper_2604_02851_b200.optim import OptimizerState, ReferenceView, StepWorkspace, step
from paper_2604_02851_b200.render import render_device

args = bench.parse()
model_h, tgt_h, poses, intr, light = bench.build_workload(args)
dm = DeviceModel.from_host(model_h, 0)
tgt = DeviceModel.from_host(tgt_h, 0)
bg = np.array([0.05, 0.05, 0.08])
views = [ReferenceView(p, intr, render_device(tgt, p, intr, light, background=bg), light, bg) for p in poses]
del tgt
lo, hi = model_h.means.min(0), model_h.means.max(0)
state = OptimizerState(dm, scene_extent=float(np.linalg.norm(hi - lo) / 2))
ws = StepWorkspace(dm)
full_np = np.arange(dm.active_count)
full_dev = torch.arange(dm.active_count, device=dm.device)
for name, sub in (("none", None), ("numpy all rows", full_np), ("device all rows", full_dev), ("none", None)):
    for _ in range(3):
        step(dm, state, views, index_subset=sub, workspace=ws, sync_loss=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(5):
        step(dm, state, views, index_subset=sub, workspace=ws, sync_loss=False)
    e1.record()
    torch.cuda.synchronize()
    print(f"{name:18s} device {e0.elapsed_time(e1) / 5:7.2f} ms  wall {(time.perf_counter() - t0) * 200:7.2f} ms")
