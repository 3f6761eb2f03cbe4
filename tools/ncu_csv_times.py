"""Print per-launch metrics from `ncu --csv --metrics ...` logs."""
import csv
import io
import sys

for f in sys.argv[1:]:
    txt = open(f).read()
    i = txt.find('"ID"')
    if i < 0:
        print(f, "no data")
        continue
    per = {}
    for r in csv.DictReader(io.StringIO(txt[i:])):
        per.setdefault(r["ID"], {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    print(f)
    for k, v in per.items():
        print(" ", k, "  ".join(f"{m.split('__')[1].split('.')[0] if '__' in m else m}={x:.4g}" for m, x in v.items()))
