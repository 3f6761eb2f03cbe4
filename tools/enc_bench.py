"""bench.py's delta-encoder and snapshot records alone (quick A/B)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.argv = sys.argv[:1]
import torch
import bench
from paper_2604_02851_b200 import _lib, synth
from paper_2604_02851_b200.model import DeviceModel
args = bench.parse()
c = _lib.ctx(0)
enc = bench.encoder_bench(c, _lib, args, torch)
dm = DeviceModel.from_host(synth.random_field(1_000_000, 3, 1920, 1080, seed=0), 0)
snap = bench.snapshot_bench(dm, torch)
print("delta", round(enc["kernel_ms_per_tick"] * 1e3, 1), "us frac", round(enc["roofline"]["frac"], 3),
      "| snapshot", round(snap["ms_per_snapshot"] * 1e3, 1), "us frac", round(snap["roofline"]["frac"], 3))
