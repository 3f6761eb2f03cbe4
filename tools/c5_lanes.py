"""Config 5 (64 viewpoints, 2M SH3, 1080p) frames/s for several lane counts."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_02851_b200 import synth
from paper_2604_02851_b200.model import DeviceModel
from paper_2604_02851_b200.render import render_device_many
m = DeviceModel.from_host(synth.random_field(2_000_000, 3, 1920, 1080, seed=7), 0)
intr, light = synth.intrinsics(1920, 1080), synth.light()
poses = synth.ring_poses(64, radius=0.6)
for lanes in (1, 2, 4, 6, 8, 12):
    outs = [torch.empty((1080, 1920, 3), dtype=torch.float32, device=m.device) for _ in range(lanes)]
    render_device_many(m, poses[:lanes], intr, light, outs=outs, lanes=lanes)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(2):
        render_device_many(m, poses, intr, light, outs=outs, lanes=lanes)
    e1.record()
    torch.cuda.synchronize()
    print(f"lanes {lanes:2d}: {128 / (e0.elapsed_time(e1) / 1e3):7.1f} frames/s")
