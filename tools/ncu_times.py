"""Summarise an `ncu --csv --metrics ...` log read from stdin: per kernel and metric, the values in launch order."""
import collections
import csv
import sys

lines = [l for l in sys.stdin if l.startswith('"')]
rows = list(csv.reader(lines))
h = rows[0]
d = collections.defaultdict(list)
for row in rows[1:]:
    if len(row) < len(h) or row[0] == "ID":
        continue
    x = dict(zip(h, row))
    try:
        d[(x["Kernel Name"][:48], x["Metric Name"])].append(float(x["Metric Value"].replace(",", "")))
    except ValueError:
        pass
step = int(sys.argv[1]) if len(sys.argv) > 1 else 1
for k, v in d.items():
    print(k, [round(a) for a in v[::step]][:24])
