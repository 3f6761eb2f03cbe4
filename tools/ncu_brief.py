"""One line per captured kernel from an ncu report: time, issue, occupancy,
DRAM bytes, top stall reasons.   python tools/ncu_brief.py gpurun_out/x.ncu-rep"""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
idx = {n: i for i, n in enumerate(h)}


SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3,
         "msecond": 1e3, "nsecond": 1e-3}
units = rows[1]


def g(r, n):
    try:
        v = float(r[idx[n]].replace(",", ""))
    except (KeyError, ValueError):
        return float("nan")
    return v * SCALE.get(units[idx[n]], 1.0)


for r in rows[2:]:
    name = r[idx["Kernel Name"]].split("(")[0][:40]
    stalls = sorted(((g(r, n), n.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""))
                     for n in h if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("ratio")), reverse=True)
    print(f"{name:40s} {g(r, 'gpu__time_duration.sum'):8.1f} us  issue {g(r, 'smsp__issue_active.avg.pct_of_peak_sustained_active'):5.1f}%  "
          f"occ {g(r, 'sm__warps_active.avg.pct_of_peak_sustained_active'):5.1f}%  regs {g(r, 'launch__registers_per_thread'):.0f}  "
          f"dram {(g(r, 'dram__bytes_read.sum') + g(r, 'dram__bytes_write.sum')) / 1e6:7.1f} MB  "
          f"inst {g(r, 'smsp__inst_executed.sum') / 1e6:7.1f}M  thr/inst {g(r, 'smsp__thread_inst_executed_per_inst_executed.ratio'):4.1f}  "
          + " ".join(f"{n}={v:.2f}" for v, n in stalls[:4]))
