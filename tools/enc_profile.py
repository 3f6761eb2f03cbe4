"""Standalone per-frame delta tick (bench.py's encoder workload) for ncu:
3 warm-up ticks, then `--ticks` ticks.  ncu -k regex:k_tick -s 9 -c 3."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2604_02851_b200 import synth  # noqa: E402
from paper_2604_02851_b200.model import DeviceModel  # noqa: E402
from paper_2604_02851_b200.protocol import DeltaTicker, PayloadBuffer  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--rows", type=int, default=2_000_000)
ap.add_argument("--ticks", type=int, default=2)
ap.add_argument("--flush", action="store_true", help="stream 256 MB through L2 before each tick (bench.py)")
ap.add_argument("--sparse", action="store_true", help="baselines 1e-6 off: the sparse path")
a = ap.parse_args()
dm = DeviceModel.from_host(synth.random_field(a.rows, 1, 1920, 1080, seed=3), 0)
off = 1e-6 if a.sparse else 2e-3
ref_m, ref_l = (dm.means - off).contiguous(), (dm.log_scales - off).contiguous()
bm, bl = ref_m.clone(), ref_l.clone()
tick = DeltaTicker(dm, {0: bm, 1: bl}, {k: PayloadBuffer(1 << 20, dm.device) for k in range(7)})
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dm.device) if a.flush else None
for _ in range(3 + a.ticks):
    bm.copy_(ref_m)
    bl.copy_(ref_l)
    if flush is not None:
        flush.add_(1.0)
    tick((0, 1, 3, 4))
torch.cuda.synchronize()
print("ok")
