"""Top SASS instructions of an ncu report with their dominant stall reasons.
usage: python tools/ncu_stalls.py report.ncu-rep [n]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h = rows[1]
si = h.index("Warp Stall Sampling (All Samples)")
st = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
recs = []
tot = {}
for r in rows[2:]:
    if len(r) < len(h):
        continue
    s = int(r[si] or 0)
    reasons = sorted(((int(r[i] or 0), h[i][6:]) for i in st), reverse=True)
    for v, k in reasons:
        tot[k] = tot.get(k, 0) + v
    recs.append((s, r[0][-5:], r[1].strip()[:60], reasons[:3]))
T = sum(x[0] for x in recs) or 1
print("stall totals:", ", ".join(f"{k} {v/T:.1%}" for k, v in sorted(tot.items(), key=lambda kv: -kv[1])[:10]))
for s, a, src, rs in sorted(recs, reverse=True)[:n]:
    print(f"{s/T:6.1%} {a} {src:60s} " + " ".join(f"{k}:{v}" for v, k in rs if v))
