"""Calibration: device time of plain streaming kernels over the encoder's
byte volumes (48 MB read, 48 MB read + 36 MB write), CUDA events, warm."""
import torch

dev = torch.device("cuda", 0)
n = 12 * 1024 * 1024  # 48 MB of float32
a = torch.randn(n, device=dev)
b = torch.randn(n, device=dev)
c = torch.empty(n, device=dev)
flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)


def t(fn, reps=20, cold=False):
    ev = []
    for _ in range(reps):
        if cold:
            flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        ev.append((e0, e1))
    torch.cuda.synchronize()
    return sorted(x.elapsed_time(y) for x, y in ev)[reps // 2] * 1e3


for cold in (False, True):
    print("cold" if cold else "warm",
          "sum48MB %.1f us" % t(lambda: a.sum(), cold=cold),
          "copy48MB %.1f us" % t(lambda: c.copy_(a), cold=cold),
          "add(a,b)->c 144MB %.1f us" % t(lambda: torch.add(a, b, out=c), cold=cold))
