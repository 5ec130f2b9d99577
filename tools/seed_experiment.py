"""Seed sample count vs seed time, survivors and scan time (C4 shape)."""
import sys, os, torch
sys.path.insert(0, '.')
import synthgen, paper_2006_08861_b200 as ol
spec = synthgen.CONFIGS["C4"].spec
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
dev = torch.device("cuda", 0)
F, C = synthgen.db_device(spec, 0, n, dev)
Q, _ = synthgen.render_device(spec, synthgen.query_points(spec, 4242, 1024), dev)
e = ol.Engine(0)
import os
if os.environ.get("TCK"): e.set_option("tc_k", int(os.environ["TCK"]))
e.upload(F, C, [n], spec.grid())
if os.environ.get("CHUNK"): e.set_option("chunk", int(os.environ["CHUNK"]))
if os.environ.get("PAIR"): e.set_option("pair", int(os.environ["PAIR"]))
if os.environ.get("CLUSTER"): e.set_option("cluster", int(os.environ["CLUSTER"]))
if os.environ.get("TCSEED"): e.set_option("tc_seed", int(os.environ["TCSEED"]))
Q3 = Q.view(-1, 1, 64)
for S in [int(x) for x in sys.argv[2].split(',')]:
    e.set_option("seed_samples", S)
    for _ in range(2): e.query(Q3, N=15)
    torch.cuda.synchronize()
    e.set_option("time_kernels", 1)
    R = 5
    for _ in range(R): e.query(Q3, N=15)
    torch.cuda.synchronize()
    t = {k: e.stat(f"time_{k}_ns") / R / 1e6 for k in ("seed", "scan", "merge", "final")}
    e.set_option("time_kernels", 0)
    print(f"pair={os.environ.get('PAIR')} samples={S} seed {t['seed']:.3f} scan {t['scan']:.3f} merge {t['merge']:.3f} final {t['final']:.3f} total {sum(t.values()):.3f} ms items {e.stat('items')} survivors/pair {e.stat('survivors')/e.stat('pairs'):.2e}")
