"""Device time per profile-0 snapshot (1M rows SH3, raw, baseline outputs),
L2 flushed before each: median over reps (bench.py snapshot_bench)."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_02851_b200 import synth  # noqa: E402
from paper_2604_02851_b200.model import DeviceModel  # noqa: E402
from paper_2604_02851_b200.protocol import PayloadBuffer, encode_snapshot_device  # noqa: E402

dm = DeviceModel.from_host(synth.random_field(1_000_000, 3, 1920, 1080, seed=0), 0)
out = PayloadBuffer(1 << 20, dm.device)
bm, bl = torch.empty_like(dm.means), torch.empty_like(dm.log_scales)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dm.device)
clean = torch.zeros(64 * 1024 * 1024, dtype=torch.float32, device=dm.device)
mode = sys.argv[1] if len(sys.argv) > 1 else "dirty"
ts = []
for i in range(23):
    flush.add_(1.0)
    if mode == "clean":  # then a read-only pass: L2 holds clean lines, no write-back left for the timed call
        clean.sum()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if "sleep" in sys.argv:  # the device waits ~100 us so the host has queued the whole call before e0 runs
        torch.cuda._sleep(200_000)
    e0.record()
    encode_snapshot_device(dm, 0, out, bm, bl)
    e1.record()
    torch.cuda.synchronize()
    if i >= 3:
        ts.append(e0.elapsed_time(e1) * 1e3)
print(f"{mode} snapshot us: median {statistics.median(ts):.1f} min {min(ts):.1f} -> {282e6 / (statistics.median(ts) * 1e-6) / 1e9:.0f} GB/s")
