"""Per-step device time of bench.py's e2e loop (host GT + loss + delta frames):
which steps are slow when the e2e number drops?"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_02851_b200 import synth  # noqa: E402
from paper_2604_02851_b200.model import DeviceModel  # noqa: E402
from paper_2604_02851_b200.optim import OptimizerState, ReferenceView, StepWorkspace, step  # noqa: E402
from paper_2604_02851_b200.protocol import DELTA_ORDER, DeltaTicker, PayloadBuffer  # noqa: E402
from paper_2604_02851_b200.render import render_device  # noqa: E402

n, V, W, H = 1_000_000, 8, 1920, 1080
model = synth.random_field(n, 3, W, H, seed=0)
tgt = synth.target_model(model, seed=1)
poses, intr, light = synth.ring_poses(V), synth.intrinsics(W, H), synth.light()
dm = DeviceModel.from_host(model, 0)
td = DeviceModel.from_host(tgt, 0)
bg = np.array([0.05, 0.05, 0.08])
gts = [render_device(td, p, intr, light, background=bg) for p in poses]
hv = [ReferenceView(p, intr, g.cpu().pin_memory(), light, bg) for p, g in zip(poses, gts)]
state = OptimizerState(dm, scene_extent=10.0, device=torch.device("cuda", 0))
ws = StepWorkspace(dm)
tick = DeltaTicker(dm, {0: dm.means.clone(), 1: dm.log_scales.clone()}, {k: PayloadBuffer(1 << 20, dm.device) for k in range(7)})
periods = {0: 1, 1: 1, 2: 10, 3: 1, 4: 1, 5: 30}
frames = "--noframes" not in sys.argv
nodelta = "--nodelta" in sys.argv
pend = None
evs = []
for i in range(40):
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    t0 = time.perf_counter()
    step(dm, state, hv, workspace=ws, sync_loss=False)
    t1 = time.perf_counter()
    if not nodelta:
        due = [int(a) for a in DELTA_ORDER if i % periods[int(a)] == 0]
        tick(due)
        done, pend = pend, tick.read_async(due, frame_epoch=1 if frames else None)
        if done is not None:
            done.result(copy=False)
    t2 = time.perf_counter()
    evs.append((e, (t1 - t0) * 1e3, (t2 - t1) * 1e3))
torch.cuda.synchronize()
for i in range(len(evs) - 1):
    print(i, round(evs[i][0].elapsed_time(evs[i + 1][0]), 2), "host step %.2f tick %.2f" % (evs[i][1], evs[i][2]))
