"""Per-frame delta tick (means, log_scales, opacity, DC) on a 1M-row model, for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2604_02851_b200 import synth
    from paper_2604_02851_b200.model import DeviceModel
    from paper_2604_02851_b200.protocol import PayloadBuffer, delta_tick_device
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 2_000_000
    deg = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    torch.cuda.set_device(0)
    dm = DeviceModel.from_host(synth.random_field(n, deg, seed=0))
    ref = {0: (dm.means - 2e-3).contiguous(), 1: (dm.log_scales - 2e-3).contiguous()}
    base = {k: v.clone() for k, v in ref.items()}
    bufs = {k: PayloadBuffer(1 << 20, dm.device) for k in range(7)}
    for _ in range(3):
        base[0].copy_(ref[0])
        base[1].copy_(ref[1])
        delta_tick_device(dm, (0, 1, 3, 4), base, bufs)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
