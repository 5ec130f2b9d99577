"""Seed variants at 1,024 frames (C4-shaped DB of argv[1] rows): the exact sampled seed (NK3,
default), the tensor-core bound pre-pass (tc_seed 1) and both (tc_seed 2)."""
import sys, torch
sys.path.insert(0, '.')
import synthgen, paper_2006_08861_b200 as ol
spec = synthgen.CONFIGS["C4"].spec
n = int(sys.argv[1]) if len(sys.argv) > 1 else 12_500_000
dev = torch.device("cuda", 0)
F, C = synthgen.db_device(spec, 0, n, dev)
e = ol.Engine(0)
e.upload(F, C, [n], spec.grid())
del F, C
Q, _ = synthgen.render_device(spec, synthgen.query_points(spec, 4242, 1024), dev)
Q3 = Q.view(-1, 1, 64)
for rep in range(2):
    for ts in (0, 1, 2):
        e.set_option("tc_seed", ts)
        for _ in range(3): e.query(Q3, N=15)
        torch.cuda.synchronize()
        e.set_option("time_kernels", 1)
        for _ in range(5): e.query(Q3, N=15)
        torch.cuda.synchronize()
        t = {k: e.stat(f"time_{k}_ns") / 5 / 1e6 for k in ("seed", "scan", "merge", "final")}
        e.set_option("time_kernels", 0)
        print(f"rows {n:,} tc_seed {ts}: seed {t['seed']:.3f} scan {t['scan']:.3f} sum {t['seed'] + t['scan']:.3f} ms "
              f"survivors/pair {e.stat('survivors') / e.stat('pairs'):.2e}", flush=True)
