"""Per-source-line share of executed instructions of one kernel in an ncu
report (needs --import-source on and -lineinfo).
    python tools/ncu_lines.py rep.ncu-rep [min_share_percent]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if r and r[0] == "Line No")
ie = hdr.index("Instructions Executed")
per, src, files = {}, {}, None
cur = None
for r in rows:
    if not r or r[0] in ("Line No",) or r[0].startswith("File") or r[0].startswith("Function"):
        if r and r[0] == "File Path":
            files = r[1]
        continue
    if r[0].isdigit():
        cur = (files, int(r[0]))
        src[cur] = r[1]
    try:
        v = int(r[ie])
    except (ValueError, IndexError):
        continue
    per[cur] = per.get(cur, 0) + v
tot = sum(per.values())
print("total", tot)
for k in sorted(per, key=lambda k: (str(k[0]), k[1])):
    if per[k] > tot * thr / 100:
        print(f"{str(k[0]).split('/')[-1]:>16}:{k[1]:<5} {per[k] / tot * 100:5.1f}%  {src.get(k, '')[:100]}")
