import numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_2604_02851_b200 import synth
from paper_2604_02851_b200.model import DeviceModel
from paper_2604_02851_b200.optim import StepWorkspace, backward_device, chain_views, ReferenceView, split_flat
from paper_2604_02851_b200.render import _subset_tensor, render_device
degree = int(sys.argv[1]) if len(sys.argv) > 1 else 3
W, H = 256, 144
host = synth.random_field(40_000, degree, W, H, seed=5)
host.active_count = 38_000
dm = DeviceModel.from_host(host, 0)
tgt = DeviceModel.from_host(synth.target_model(host, seed=6), 0)
intr = synth.intrinsics(W, H); light = synth.light(); poses = synth.ring_poses(5, radius=1.5)
views = [ReferenceView(p, intr, render_device(tgt, p, intr, light), light, np.zeros(3)) for p in poses]
rng = np.random.default_rng(0)
for subset in (None, np.sort(rng.choice(40_000, 25_000, replace=False))):
    sub = _subset_tensor(subset, dm.device)
    ws = StepWorkspace(dm)
    n_grad = dm.active_count * (11 + 3 * (degree + 1) ** 2)
    g_ref = torch.zeros(n_grad, dtype=torch.float32, device=dm.device)
    loss = torch.zeros(1, dtype=torch.float64, device=dm.device)
    for v in views:
        backward_device(dm, v, g_ref, loss, subset_tensor=sub)
    n_in = int(sub.numel()) if sub is not None else dm.count
    g9, rinv = ws.defer_buffers(len(views), n_in, dm.device)
    g_def = torch.zeros_like(g_ref)
    for i, v in enumerate(views):
        backward_device(dm, v, g_def, loss, subset_tensor=sub, defer=(g9[i], rinv[i]))
    chain_views(dm, views, g9, rinv, g_def, sub)
    a = split_flat(g_ref, dm.active_count, degree); b = split_flat(g_def, dm.active_count, degree)
    for k in a:
        d = (a[k] != b[k])
        n = int(d.sum())
        if n:
            idx = torch.nonzero(d.reshape(d.shape[0], -1).any(1)).flatten()
            print("subset" if subset is not None else "full", k, "differ", n, "rows", idx[:10].tolist(), "nrows", idx.numel())
            r = int(idx[0]); print(a[k][r].flatten()[:8].tolist()); print(b[k][r].flatten()[:8].tolist())
        else:
            print("subset" if subset is not None else "full", k, "equal")
