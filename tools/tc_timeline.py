"""Per-tile timeline of the tensor-core scan's CTA 0 (tc_debug 32 | 2048: clock64 stamps):
MMA warp past its tempty wait / done issuing + committing; the epilogue group's last warp past
tfull, its last release, its last tile end.  Prints the steady-state intervals.
  python tools/tc_timeline.py [rows]"""
import sys, torch
sys.path.insert(0, '.')
import numpy as np
import synthgen, paper_2006_08861_b200 as ol
spec = synthgen.CONFIGS["C4"].spec
n = int(sys.argv[1]) if len(sys.argv) > 1 else 20_000_000
dev = torch.device("cuda", 0)
F, C = synthgen.db_device(spec, 0, n, dev)
Q, _ = synthgen.render_device(spec, synthgen.query_points(spec, 4242, 1024), dev)
e = ol.Engine(0)
e.upload(F, C, [n], spec.grid())
del F, C
Q3 = Q.view(-1, 1, 64)
for _ in range(2): e.query(Q3, N=15)
e.set_option("tc_debug", 32 | 2048)
e.query(Q3, N=15)
torch.cuda.synchronize()
T = 120
v = np.array([e.stat(f"prof{64 + i}") for i in range(T * 8)], dtype=np.int64).reshape(T, 8)
ok = (v[:, :5] > 0).all(axis=1)
n_ok = int(np.argmin(ok)) if not ok.all() else T
v = v[:n_ok]
t0 = v[0, 0]
print(f"tiles recorded: {n_ok}")
print("  t   tempty_ok  issued   tfull_ok  release   end   events  bounds-ok  ld0-ok  (cycles from MMA tempty_ok of tile 0)")
for t in range(min(n_ok, 40)):
    print(f"{t:3d} " + " ".join(f"{x - t0:9d}" for x in v[t, :5]) + f" {v[t, 5]:6d} " + " ".join(f"{x - t0:9d}" for x in v[t, 6:8]))
print("events per tile, tiles 0-9 / 10-49 / 50-99 / 100-119:", [round(float(v[a:b, 5].mean()), 1) for a, b in ((0, 10), (10, 50), (50, 100), (100, n_ok))])
print("cycles per tile, same ranges:", [round(float(np.diff(v[a:b, 1]).mean())) for a, b in ((0, 10), (10, 50), (50, 100), (100, n_ok))])
s = slice(8, n_ok)
r = lambda a: float(np.mean(a))
tile_period = r(np.diff(v[s, 1]))
print("total cycles for the recorded tiles:", int(v[-1, 4] - t0), "; rows:", n, "; items:", e.stat("items"), "; chunk:", e.stat("chunk"))
print(f"steady state (tiles 8..{n_ok - 1}): period {tile_period:.0f} cycles/tile")
print(f"  MMA issue+commit            {r(v[s, 1] - v[s, 0]):.0f}")
print(f"  commit done -> tfull seen   {r(v[s, 2] - v[s, 1]):.0f}   (MMA execution + arrive + wake of the group's last warp)")
print(f"  tfull -> last release       {r(v[s, 3] - v[s, 2]):.0f}   (the group's TMEM reads)")
print(f"  last release -> tile end    {r(v[s, 4] - v[s, 3]):.0f}")
rel = v[:, 3]
print(f"  release(t-2) -> MMA past tempty(t): {r(v[10:n_ok, 0] - rel[8:n_ok - 2]):.0f}   (MMA warp wake)")
print(f"  tfull(t) - tfull(t-1): {r(np.diff(v[s, 2])):.0f}; release(t) - release(t-1): {r(np.diff(v[s, 3])):.0f}")
