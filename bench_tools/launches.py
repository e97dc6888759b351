"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: total ms and launch
count per kernel name."""
import csv
import sys

UNIT = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3}
rows = list(csv.reader(l for l in open(sys.argv[1]) if l.startswith('"')))
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
agg = {}
for r in rows[1:]:
    name = r[ki].replace("<unnamed>::", "").replace("void ", "").split("(")[0].split("<")[0]
    v = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1e-6)
    a = agg.setdefault(name, [0.0, 0])
    a[0] += v
    a[1] += 1
tot = sum(a[0] for a in agg.values())
for k, (v, c) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{k:40s} {v:10.3f} ms  x{c:<5d} {100 * v / tot:5.1f} %")
print(f"{'total':40s} {tot:10.3f} ms")
