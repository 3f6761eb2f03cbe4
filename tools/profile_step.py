"""One warm-up + one timed optimizer step of the bench workload, for ncu.

    python tools/profile_step.py [--n 1000000] [--views 8]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--views", type=int, default=8)
    ap.add_argument("--steps", type=int, default=2)
    args = ap.parse_args()
    import numpy as np
    import torch

    from paper_2604_02851_b200 import synth
    from paper_2604_02851_b200.model import DeviceModel
    from paper_2604_02851_b200.optim import OptimizerState, ReferenceView, StepWorkspace, step
    from paper_2604_02851_b200.protocol import PayloadBuffer, encode_delta_device
    from paper_2604_02851_b200.render import render_device

    torch.cuda.set_device(0)
    model = synth.random_field(args.n, 3, 1920, 1080, seed=0)
    dm = DeviceModel.from_host(model)
    tgt = DeviceModel.from_host(synth.target_model(model, 1))
    intr = synth.intrinsics()
    light = synth.light()
    poses = synth.ring_poses(args.views)
    views = [ReferenceView(p, intr, render_device(tgt, p, intr, light, background=synth.BACKGROUND), light,
                           synth.BACKGROUND) for p in poses]
    state = OptimizerState(dm, scene_extent=3.0)
    ws = StepWorkspace(dm)
    base = dm.means.clone()
    buf = PayloadBuffer(1 << 24, dm.device)
    for _ in range(args.steps):
        step(dm, state, views, workspace=ws, sync_loss=False)
        encode_delta_device(0, dm.means, base, base, None, buf)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
