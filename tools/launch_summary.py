"""Summarise an ncu --metrics gpu__time_duration.sum launch list (csv) per kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"ms": 1e3, "msecond": 1e3, "us": 1, "usecond": 1, "ns": 1e-3, "nsecond": 1e-3, "s": 1e6, "second": 1e6}
agg = collections.OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0]
    agg.setdefault(name, []).append(float(r[vi].replace(",", "")) * scale[r[ui]])
tot = sum(sum(v) for v in agg.values())
print(f"{'kernel':42s} {'launches':>8s} {'total_us':>12s} {'mean_us':>11s} {'share':>7s}")
for k, v in agg.items():
    print(f"{k:42s} {len(v):8d} {sum(v):12.1f} {sum(v)/len(v):11.1f} {sum(v)/tot:7.1%}")
