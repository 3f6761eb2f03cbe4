"""Utilisation of the backward blend walk on the bench workload (diagnostics build).

  SS_NVCC_EXTRA=-DSS_BWD_STATS python -m paper_2604_02851_b200._build --force
  python tools/bwd_stats.py
"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2604_02851_b200 import _lib, synth  # noqa: E402
from paper_2604_02851_b200.model import DeviceModel  # noqa: E402
from paper_2604_02851_b200.optim import OptimizerState, ReferenceView, StepWorkspace, step  # noqa: E402
from paper_2604_02851_b200.render import render_device  # noqa: E402

host = synth.random_field(1_000_000, 3, 1920, 1080, seed=0)
tgt = DeviceModel.from_host(synth.target_model(host, seed=1), 0)
dm = DeviceModel.from_host(host, 0)
poses = synth.ring_poses(8)
intr = synth.intrinsics()
light = synth.light()
bg = np.array([0.05, 0.05, 0.08])
views = [ReferenceView(p, intr, render_device(tgt, p, intr, light, background=bg), light, bg) for p in poses]
state = OptimizerState(dm, scene_extent=4.0)
ws = StepWorkspace(dm)
c = _lib.ctx(0)
out = (ctypes.c_uint64 * 8)()
for i in range(3):
    step(dm, state, views, workspace=ws)
    c.check(c.lib.ss_debug_bwd_stats(c.handle, out, 1))
s = [v / 8 for v in out]  # per view
print(f"per view: pairs {s[0]:.4g}, walked {s[1]:.4g} ({s[1]/s[0]:.1%}), with active px {s[2]:.4g} ({s[2]/s[1]:.1%} of walked)")
print(f"active (px, splat) pairs {s[3]:.4g} = {s[3]/s[2]:.1f} per active pair; body lanes/pair {s[4]/s[2]:.1f}")
print(f"pixel slots computed {s[5]:.4g}: utilisation {s[3]/s[5]:.1%}")
