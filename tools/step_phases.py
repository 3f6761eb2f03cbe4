"""Where does the 8-view step's time go under the view lanes?  Events on the
caller's stream at the phase boundaries of optim.step (views forked ->
joined -> chain rule -> Adam), averaged over steps."""
import os, sys
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
marks = []


def mark(name):
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    marks.append((name, e))


K = optim._DeviceKernels
orig = {n: getattr(K, n) for n in ("stage", "join", "chain_batch", "sum_losses", "adam")}
K.stage = lambda self, lv: (mark("start"), orig["stage"](self, lv))[1]
K.join = lambda self: (orig["join"](self), mark("views done"))[1]
K.chain_batch = lambda self, v, r: (orig["chain_batch"](self, v, r), mark("chain rule"))[1]
K.adam = lambda self, n: (orig["adam"](self, n), mark("adam"))[1]
for _ in range(3):
    step(dm, state, views, workspace=ws, sync_loss=False)
torch.cuda.synchronize()
acc = {}
steps = 10
for _ in range(steps):
    marks.clear()
    step(dm, state, views, workspace=ws, sync_loss=False)
    mark("end")
    torch.cuda.synchronize()
    for (a, ea), (b, eb) in zip(marks, marks[1:]):
        acc[f"{a} -> {b}"] = acc.get(f"{a} -> {b}", 0.0) + ea.elapsed_time(eb) / steps
tot = sum(acc.values())
for k, v in acc.items():
    print(f"{k:28s} {v:7.3f} ms")
print(f"{'total':28s} {tot:7.3f} ms -> {8 / tot * 1e3:.1f} views/s")
