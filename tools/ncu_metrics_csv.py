"""Pivot an `ncu --metrics ... --csv --log-file` launch list: one line per
launch with its metrics.   python tools/ncu_metrics_csv.py gpurun_out/x.csv"""
import csv
import sys

lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
rows = list(csv.reader(lines))
h = rows[0]
ki, ii, mi, vi, ui = (h.index(k) for k in ("Kernel Name", "ID", "Metric Name", "Metric Value", "Metric Unit"))
launches = {}
for r in rows[1:]:
    d = launches.setdefault(r[ii], {"name": r[ki].split("(")[0][:44]})
    d[r[mi]] = (r[vi], r[ui])
for i, d in sorted(launches.items(), key=lambda x: int(x[0])):
    print(f"{i:>4} {d.pop('name'):44s} " + "  ".join(f"{k.split('.')[0].split('__')[-1]}={v} {u}" for k, (v, u) in d.items()))
