"""Device CRC-32 of a 26 MB payload (the raw per-frame delta set at 2M rows)
vs host zlib.crc32."""
import os
import sys
import time
import zlib

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_02851_b200.protocol import crc32_device  # noqa: E402

n = 26_000_064
d = torch.randint(0, 256, (n,), dtype=torch.uint8, device="cuda")
for _ in range(3):
    crc32_device(d)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    c = crc32_device(d)
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) / 20 * 1e3
h = d.cpu().numpy().tobytes()
t = time.perf_counter()
ref = zlib.crc32(h)
hs = time.perf_counter() - t
assert ref == int(c.item()) & 0xFFFFFFFF
print(f"device crc32 {us:.1f} us ({n / us / 1e3:.1f} GB/s); host zlib.crc32 {hs * 1e3:.2f} ms")
