"""Summarise an ncu launch list (csv; gpu__time_duration.sum and optionally dram bytes)
per kernel: launches, total / mean time, share of the time, DRAM bytes per launch."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
tscale = {"ms": 1e3, "msecond": 1e3, "us": 1, "usecond": 1, "ns": 1e-3, "nsecond": 1e-3, "s": 1e6, "second": 1e6}
bscale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
t = collections.OrderedDict()
b = collections.defaultdict(float)
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0]
    v = float(r[vi].replace(",", ""))
    if r[mi] == "gpu__time_duration.sum":
        t.setdefault(name, []).append(v * tscale[r[ui]])
    elif r[mi].startswith("dram__bytes"):
        b[name] += v * bscale[r[ui]]
tot = sum(sum(v) for v in t.values())
print(f"{'kernel':42s} {'launches':>8s} {'total_us':>12s} {'mean_us':>11s} {'share':>7s} {'dram_GB/launch':>15s}")
for k, v in t.items():
    print(f"{k:42s} {len(v):8d} {sum(v):12.1f} {sum(v)/len(v):11.1f} {sum(v)/tot:7.1%} {b[k]/len(v)/1e9:15.3f}")
