"""Delta tick per-frame set (bench encoder_bench) with SH DC read through the
(N, 3, B) rows vs from a contiguous (N, 3) column: how much does the DC
layout cost?   python tools/dc_probe.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2604_02851_b200 import _lib, synth
from paper_2604_02851_b200.model import DeviceModel
from paper_2604_02851_b200.protocol import DeltaTicker, PayloadBuffer

c = _lib.ctx(0)
n = 2_000_000
dm = DeviceModel.from_host(synth.random_field(n, 1, 1920, 1080, seed=3), 0)
a = dm.active_count
per_frame = (0, 1, 3, 4)
ref_m = (dm.means - 2e-3).contiguous()
ref_l = (dm.log_scales - 2e-3).contiguous()
bm, bl = ref_m.clone(), ref_l.clone()
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dm.device)
clean = torch.zeros(64 * 1024 * 1024, dtype=torch.float32, device=dm.device)
dc = dm.sh_coeffs.reshape(n, 3, -1)[:, :, 0].contiguous()


def run(mirror, reps=30):
    bufs = {k: PayloadBuffer(1 << 20, dm.device) for k in range(7)}
    tick = DeltaTicker(dm, {0: bm, 1: bl}, bufs)
    if mirror:
        orig = tick._build

        def build(attrs):
            jobs = orig(attrs)
            for i, at in enumerate(attrs):
                if int(at) == 4:
                    j = jobs[i]
                    j.cur, j.row_stride, j.inner, j.outer, j.col0 = dc.data_ptr(), 3, 1, 1, 0
            return jobs
        tick._build = build
    for _ in range(3):
        tick(per_frame)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        bm.copy_(ref_m)
        bl.copy_(ref_l)
        flush.add_(1.0)
        clean.sum()  # bench.l2_flush: no dirty lines of the flush left
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        tick(per_frame)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ts.sort()
    return ts[len(ts) // 2] * 1e3, bytes(bufs[4].data[:int(bufs[4].length.item())].cpu().numpy())


t0, p0 = run(False)
t1, p1 = run(True)
print(f"DC through rows {t0:.1f} us, DC column {t1:.1f} us, payload equal {p0 == p1}")
t0, _ = run(False)
print(f"DC through rows again {t0:.1f} us")
