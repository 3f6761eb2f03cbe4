"""Summarise ncu outputs for profiles/.

  python tools/ncu_summary.py launches <launches.csv> > profiles/<round>_launches_summary.txt
  python tools/ncu_summary.py report <file.ncu-rep> > profiles/<round>_kernels_ncu.txt
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "time"),
    ("smsp__inst_executed.sum", "warp_instr"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem_%peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_%peak"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1_%"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma_pipe_%"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64_pipe_%"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "threads/warp_instr"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        name = d["Kernel Name"].split("(")[0].replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
        v = float(d["Metric Value"]) * {"nsecond": 1, "usecond": 1e3, "msecond": 1e6}.get(d["Metric Unit"], 1)
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    print("# ncu --metrics gpu__time_duration.sum --clock-control none (cold cache, serialised: compare shares)")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k[:64]:64s} launches={v[0]:5d} total_ms={v[1] / 1e6:9.3f} share={v[1] / tot * 100:5.1f}%")
    print(f"total_ms {tot / 1e6:.3f}")


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    print("# ncu --set full --clock-control none, one launch per line (units in header)")
    cols = [(k, n) for k, n in KEYS if k in h]
    print("kernel | " + " | ".join(f"{n} [{units[h.index(k)]}]" for k, n in cols))
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0].replace("<unnamed>::", "")
        print(name + " | " + " | ".join(r[h.index(k)] for k, _ in cols))


if __name__ == "__main__":
    {"launches": launches, "report": report}[sys.argv[1]](sys.argv[2])
