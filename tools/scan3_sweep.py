"""CUDA-core small-batch kernels: scan2 (row-pair streaming, default) vs scan3 (TMA-fed,
option scan2 = 2), tensor-core filter off, C4-shaped DB prefixes and 1-8 frames."""
import sys, torch
sys.path.insert(0, '.')
import synthgen, paper_2006_08861_b200 as ol
spec = synthgen.CONFIGS["C4"].spec
dev = torch.device("cuda", 0)
for n in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1000000,10000000,100000000").split(",")]:
    F, C = synthgen.db_device(spec, 0, n, dev)
    e = ol.Engine(0)
    e.set_option("tc", 0)
    e.upload(F, C, [n], spec.grid())
    del F, C
    for B in (1, 2, 4, 8):
        Q, _ = synthgen.render_device(spec, synthgen.query_points(spec, 4242, B), dev)
        Q3 = Q.view(-1, 1, 64)
        res = []
        for v in (1, 2, 1, 2):
            e.set_option("scan2", v)
            for _ in range(3): e.query(Q3, N=15)
            torch.cuda.synchronize()
            e.set_option("time_kernels", 1)
            for _ in range(10): e.query(Q3, N=15)
            torch.cuda.synchronize()
            ms = e.stat("time_scan_ns") / 10 / 1e6
            for k in ("seed", "merge", "final"): e.stat(f"time_{k}_ns")
            e.set_option("time_kernels", 0)
            res.append(ms)
        print(f"rows {n:>11,} frames {B}: scan2 {min(res[0], res[2]):.3f}  scan3 {min(res[1], res[3]):.3f} ms  "
              f"(coarse plane {n * 64 / 1e9:.2f} GB: {n * 64 / min(res[1], res[3]) / 1e6:.0f} GB/s scan3)", flush=True)
    e.close()
    torch.cuda.empty_cache()
