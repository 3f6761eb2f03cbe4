"""Snapshot encode (1M rows, SH3, profile 0 raw) x3 for ncu launch lists."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_02851_b200 import synth  # noqa: E402
from paper_2604_02851_b200.model import DeviceModel  # noqa: E402
from paper_2604_02851_b200.protocol import PayloadBuffer, encode_snapshot_device  # noqa: E402

dm = DeviceModel.from_host(synth.random_field(1_000_000, 3, 1920, 1080, seed=0), 0)
out = PayloadBuffer(1 << 20, dm.device)
bm, bl = torch.empty_like(dm.means), torch.empty_like(dm.log_scales)
for _ in range(3):
    encode_snapshot_device(dm, 0, out, bm, bl)
torch.cuda.synchronize()
print("ok")
