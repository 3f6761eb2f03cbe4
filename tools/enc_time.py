"""Device time per delta tick, bench.py's encoder workload (2M rows, per-frame
set, dense residual, 256 MB L2 flush between ticks): median over reps."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2604_02851_b200 import synth  # noqa: E402
from paper_2604_02851_b200.model import DeviceModel  # noqa: E402
from paper_2604_02851_b200.protocol import DeltaTicker, PayloadBuffer  # noqa: E402

sparse = "--sparse" in sys.argv
dm = DeviceModel.from_host(synth.random_field(2_000_000, 1, 1920, 1080, seed=3), 0)
off = 1e-6 if sparse else 2e-3
ref_m, ref_l = (dm.means - off).contiguous(), (dm.log_scales - off).contiguous()
bm, bl = ref_m.clone(), ref_l.clone()
tick = DeltaTicker(dm, {0: bm, 1: bl}, {k: PayloadBuffer(1 << 20, dm.device) for k in range(7)})
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dm.device)
ts = []
for i in range(43):
    bm.copy_(ref_m)
    bl.copy_(ref_l)
    flush.add_(1.0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    tick((0, 1, 3, 4))
    e1.record()
    torch.cuda.synchronize()
    if i >= 3:
        ts.append(e0.elapsed_time(e1) * 1e3)
print(f"{'sparse' if sparse else 'dense'} tick us: median {statistics.median(ts):.1f} min {min(ts):.1f}")
