"""Seed cost vs scan at small batches (C4 database): seed / scan ms and survivors for the
automatic seed (two kernels), the one-CTA-per-job seed (seed_kernel 0) and fewer samples.
  python tools/seed_small.py [rows]"""
import sys, torch
sys.path.insert(0, '.')
import synthgen, paper_2006_08861_b200 as ol
spec = synthgen.CONFIGS["C4"].spec
n = int(sys.argv[1]) if len(sys.argv) > 1 else spec.n_entries
dev = torch.device("cuda", 0)
F, C = synthgen.db_device(spec, 0, n, dev)
e = ol.Engine(0)
e.upload(F, C, [n], spec.grid())
del F, C
for nq in (8, 64, 256):
    Q, _ = synthgen.render_device(spec, synthgen.query_points(spec, 4242, nq), dev)
    Q3 = Q.view(-1, 1, 64)
    for name, opts in (("auto", {}), ("1-kernel", {"seed_kernel": 0}), ("S=2048", {"seed_samples": 2048}),
                       ("S=1024", {"seed_samples": 1024}), ("1k S=2048", {"seed_kernel": 0, "seed_samples": 2048})):
        e.set_option("seed_kernel", 1); e.set_option("seed_samples", 0)
        for k, v in opts.items(): e.set_option(k, v)
        for _ in range(3): e.query(Q3, N=15)
        torch.cuda.synchronize()
        e.set_option("time_kernels", 1)
        reps = 10
        for _ in range(reps): e.query(Q3, N=15)
        torch.cuda.synchronize()
        t = {k: e.stat(f"time_{k}_ns") / reps / 1e6 for k in ("seed", "scan", "merge", "final")}
        e.set_option("time_kernels", 0)
        print(f"rows {n:,} frames {nq:4d} {name:10s} seed {t['seed']:.3f} scan {t['scan']:.3f} merge {t['merge']:.3f} "
              f"final {t['final']:.3f} ms  survivors/pair {e.stat('survivors') / e.stat('pairs'):.2e}", flush=True)
