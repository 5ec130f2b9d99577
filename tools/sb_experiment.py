"""Small-batch (HBM regime) scan timing on the C4 DB prefix."""
import sys, torch
sys.path.insert(0, '.')
import synthgen, paper_2006_08861_b200 as ol
spec = synthgen.CONFIGS["C4"].spec
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
B = int(sys.argv[2]) if len(sys.argv) > 2 else 8
dev = torch.device("cuda", 0)
F, C = synthgen.db_device(spec, 0, n, dev)
Q, _ = synthgen.render_device(spec, synthgen.query_points(spec, 4242, B), dev)
e = ol.Engine(0)
e.set_option("tc", 0)
e.upload(F, C, [n], spec.grid())
del F, C
Q3 = Q.view(-1, 1, 64)
for opts in ([("scan2", 2)], [("scan2", 1)], [("scan2", 0)]):
    for k, v in opts: e.set_option(k, v)
    for _ in range(3): e.query(Q3, N=15)
    torch.cuda.synchronize()
    e.set_option("time_kernels", 1)
    for _ in range(10): e.query(Q3, N=15)
    torch.cuda.synchronize()
    ms = e.stat("time_scan_ns") / 10 / 1e6
    for k in ("seed", "merge", "final"): e.stat(f"time_{k}_ns")
    e.set_option("time_kernels", 0)
    print(f"{opts} scan {ms:.3f} ms = {n*64/ms/1e6:.0f} GB/s coarse; survivors/pair {e.stat('survivors')/e.stat('pairs'):.2e} items {e.stat('items')} chunk {e.stat('chunk')}")
