"""Seed sample count vs seed + scan time (C4-shaped database of argv[1] rows, NQ frames).
  NQ=1024 python tools/seed_samples.py 1000000 2048,4096,8192,16384"""
import os, sys, torch
sys.path.insert(0, '.')
import synthgen, paper_2006_08861_b200 as ol
spec = synthgen.CONFIGS["C4"].spec
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
nq = int(os.environ.get("NQ", 1024))
dev = torch.device("cuda", 0)
F, C = synthgen.db_device(spec, 0, n, dev)
e = ol.Engine(0)
e.upload(F, C, [n], spec.grid())
del F, C
Q, _ = synthgen.render_device(spec, synthgen.query_points(spec, 4242, nq), dev)
Q3 = Q.view(-1, 1, 64)
for S in [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "0,2048,4096,8192,16384").split(",")]:
    e.set_option("seed_samples", S)
    for _ in range(3): e.query(Q3, N=15)
    torch.cuda.synchronize()
    e.set_option("time_kernels", 1)
    reps = 10
    for _ in range(reps): e.query(Q3, N=15)
    torch.cuda.synchronize()
    t = {k: e.stat(f"time_{k}_ns") / reps / 1e6 for k in ("seed", "scan", "merge", "final")}
    e.set_option("time_kernels", 0)
    print(f"rows {n:,} frames {nq} samples {S or 'auto':>5}: seed {t['seed']:.3f} scan {t['scan']:.3f} "
          f"seed+scan {t['seed'] + t['scan']:.3f} ms  survivors/pair {e.stat('survivors') / e.stat('pairs'):.2e}", flush=True)
