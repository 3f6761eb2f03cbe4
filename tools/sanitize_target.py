"""A small workload for compute-sanitizer: one optimizer step (preprocess,
depth + tile onesweep sorts, binning, k_blend_fwd2, k_blend_bwd both modes,
partial sums, chain rule, Adam) and one delta tick (k_tick_fused with dense,
sparse and absolute jobs)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2604_02851_b200 import synth  # noqa: E402
from paper_2604_02851_b200.model import DeviceModel  # noqa: E402
from paper_2604_02851_b200.optim import OptimizerState, ReferenceView, StepWorkspace, step  # noqa: E402
from paper_2604_02851_b200.protocol import DeltaTicker, PayloadBuffer  # noqa: E402
from paper_2604_02851_b200.render import render_device  # noqa: E402

W, H = 192, 128
host = synth.random_field(12_000, 3, W, H, seed=1)
dm = DeviceModel.from_host(host, 0)
tgt = DeviceModel.from_host(synth.target_model(host, seed=2), 0)
intr = synth.intrinsics(W, H)
light = synth.light()
views = [ReferenceView(p, intr, render_device(tgt, p, intr, light), light, np.zeros(3)) for p in synth.ring_poses(2)]
state = OptimizerState(dm, scene_extent=2.0)
ws = StepWorkspace(dm)
step(dm, state, views, workspace=ws)
step(dm, state, views, workspace=ws, deterministic=False)
a = dm.active_count
bm = (dm.means - 2e-3).contiguous()
bl = dm.log_scales.clone()
bl[::7] -= 0.01
tick = DeltaTicker(dm, {0: bm, 1: bl}, {k: PayloadBuffer(1 << 16, dm.device) for k in range(7)})
tick((0, 1, 2, 3, 4, 5))
torch.cuda.synchronize()
print("sanitize target ok")
