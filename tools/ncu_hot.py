"""Top source lines / SASS of an ncu report by warp-stall samples.
usage: python tools/ncu_hot.py report.ncu-rep [n]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur_file = None; lines = []; sass = []
hdr = None
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]; continue
    if r and r[0] == "Line No":
        hdr = r; continue
    if hdr is None or len(r) < 5:
        continue
    try:
        samp = int(r[4]); ex = int(r[7] or 0)
    except ValueError:
        continue
    if r[0]:
        lines.append((samp, f"{cur_file}:{r[0]}", r[1][:90], ex))
    else:
        sass.append((samp, r[3][:70], ex))
tot = sum(s for s, *_ in lines) or 1
print(f"total samples {tot}")
for s, loc, src, ex in sorted(lines, reverse=True)[:n]:
    print(f"{s/tot:6.1%} {loc:22s} {src}")
print("--- sass")
for s, ins, ex in sorted(sass, reverse=True)[:n]:
    print(f"{s/tot:6.1%} {ins:70s} exec={ex}")
