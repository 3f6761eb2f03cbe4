"""bench.py's live server tick, stage by stage with a device sync between
stages (where do the 30 ms go?)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.argv = sys.argv[:1]
import numpy as np
import torch
import bench
from paper_2604_02851_b200 import engine, pool
from paper_2604_02851_b200.model import DeviceModel
from paper_2604_02851_b200.optim import OptimizerState, ReferenceView, StepWorkspace, step
from paper_2604_02851_b200.protocol import DELTA_ORDER, DeltaTicker, PayloadBuffer
from paper_2604_02851_b200.render import update_light_visibility
from paper_2604_02851_b200.scene import scene_from_dict

args = bench.parse()
model_h, tgt_h, poses, intr, light = bench.build_workload(args)
dm = DeviceModel.from_host(model_h, 0)
lo, hi = model_h.means.min(0), model_h.means.max(0)
state = OptimizerState(dm, scene_extent=float(np.linalg.norm(hi - lo) / 2))
scene = scene_from_dict(bench.ENGINE_SCENE)
gts = [torch.empty((intr.height, intr.width, 3), dtype=torch.float32, device=dm.device) for _ in poses]
views = [ReferenceView(p, intr, g, light, np.zeros(3)) for p, g in zip(poses, gts)]
lcam = engine.build_light_camera(np.array([-5.0, -1.0, -1.0]), np.array([5.0, 3.0, 9.0]), light.direction, 256)
rig, rintr = engine.build_dome_rig(np.array([0.0, 0.3, 0.0]), 0.4, 4, 3.0, width=256, height=256, fov_y=1.3)
grid = pool.GridIndex(cell_size=0.5, origin=(0.0, 0.0, 0.0))
ws = StepWorkspace(dm)
acc = {}


def t(name, fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    acc[name] = acc.get(name, 0.0) + (time.perf_counter() - t0) * 1e3
    return r


for i in range(8):
    if i == 2:
        acc.clear()
    ld = t("light depth", lambda: engine.render_ortho_depth(scene, lcam, as_tensor=True))
    t("light vis", lambda: update_light_visibility(dm, ld, lcam))
    bufs = t("capture x4", lambda: [engine.capture_input_buffers(scene, p, rintr, as_tensors=True) for p in rig])
    t("cull+init", lambda: engine.init_gaussians(engine.cull_input_samples(bufs, as_tensors=True),
                                                 sh_degree=dm.sh_degree, as_device=True))
    t("gt x8", lambda: [engine.render_ground_truth_device(scene, p, intr, out=g) for p, g in zip(poses, gts)])
    sub = t("precull", lambda: pool.precull(dm, grid, poses, intr, as_tensor=True) if grid.cells is not None else None)
    t("step", lambda: step(dm, state, views, index_subset=sub, workspace=ws, sync_loss=False))
    t("grid rebuild", lambda: grid.rebuild(dm))
    t("freeze policy", lambda: pool.freeze_policy(dm, state, age_threshold=120, grad_threshold=3e-4))
n = 6
for k, v in acc.items():
    print(f"{k:16s} {v / n:8.3f} ms")
print(f"{'total':16s} {sum(acc.values()) / n:8.3f} ms")
