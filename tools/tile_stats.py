import sys, numpy as np
sys.path.insert(0, '.')
from paper_2604_02851_b200 import synth
from paper_2604_02851_b200.render import tile_bins
m = synth.random_field(1_000_000, 3, 1920, 1080, seed=0)
intr = synth.intrinsics(1920, 1080)
for v, pose in enumerate(synth.ring_poses(8)[:3]):
    rows, ranges, ranks = tile_bins(m, pose, intr)
    cnt = ranges[:, 1] - ranges[:, 0]
    print(v, "pairs", cnt.sum(), "tiles", len(cnt), "mean", cnt.mean(), "p50", np.percentile(cnt, 50), "p99", np.percentile(cnt, 99), "max", cnt.max(), ">2048:", (cnt > 2048).sum(), ">4096:", (cnt > 4096).sum())
