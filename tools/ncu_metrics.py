"""Print (launch id, grid, metric, value) rows of an ncu --csv --metrics log."""
import csv
import sys

for path in sys.argv[1:]:
    rows = [ln for ln in open(path) if ln.startswith('"')]
    for r in csv.DictReader(rows):
        print(r["ID"], r["Grid Size"], r["Metric Name"], r["Metric Value"])
