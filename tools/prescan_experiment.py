"""Threshold pre-scan experiment (option "prescan", per mille of rows; the option was removed
after this measurement, DESIGN.md §11 "Tried and measured"): seed + scan time, survivors,
and identical top-N vs prescan = 0, at C3 / C4 shapes (1,024 frames, N = 15)."""
import sys, torch
import numpy as np
sys.path.insert(0, '.')
import synthgen, paper_2006_08861_b200 as ol
spec = synthgen.CONFIGS["C4"].spec
dev = torch.device("cuda", 0)
for n in [int(x) for x in sys.argv[1].split(',')]:
    F, C = synthgen.db_device(spec, 0, n, dev)
    Q, _ = synthgen.render_device(spec, synthgen.query_points(spec, 4242, 1024), dev)
    e = ol.Engine(0)
    e.upload(F, C, [n], spec.grid())
    Q3 = Q.view(-1, 1, 64)
    base = None
    for P in [int(x) for x in sys.argv[2].split(',')]:
        e.set_option("prescan", P)
        for _ in range(2): e.query(Q3, N=15)
        torch.cuda.synchronize()
        got = e.topk()
        if base is None: base = got
        same = np.array_equal(got.view(np.uint8), base.view(np.uint8))
        e.set_option("time_kernels", 1)
        R = 5
        for _ in range(R): e.query(Q3, N=15)
        torch.cuda.synchronize()
        t = {k: e.stat(f"time_{k}_ns") / R / 1e6 for k in ("seed", "scan", "merge", "final")}
        e.set_option("time_kernels", 0)
        print(f"rows={n} prescan={P} seed {t['seed']:.3f} scan {t['scan']:.3f} total {sum(t.values()):.3f} ms "
              f"survivors/pair {e.stat('survivors')/e.stat('pairs'):.2e} identical={same}", flush=True)
    del F, C, e
    torch.cuda.empty_cache()
