"""C3 (1M-row campus DB, 1,024 query frames, N = 15, Alg. 2 on) swept over the subspace count
n_s in {1, 5, 50} (equal consecutive splits of the DB) and the coarse width K_c in
{0, 8, 16, 32}: device ms per step (CUDA events over 10 steps) and the
stage split.  The tensor-core filter is automatic (1,024 frames: on)."""
import sys, torch
sys.path.insert(0, '.')
import numpy as np
import synthgen, paper_2006_08861_b200 as ol
cfg = synthgen.CONFIGS["C3"]; spec = cfg.spec
n = spec.n_entries
dev = torch.device("cuda", 0)
F, C = synthgen.db_device(spec, 0, n, dev)
Q, _ = synthgen.render_device(spec, synthgen.query_points(spec, 4242, 1024), dev)
Q3 = Q.view(-1, 1, 64)
for ns in (1, 5, 50):
    sizes = [n // ns + (1 if i < n % ns else 0) for i in range(ns)]
    for kc in (0, 8, 16, 32):
        e = ol.Engine(0, coarse_k=kc)
        e.upload(F, C, sizes, spec.grid())
        for _ in range(3): e.query(Q3, N=15, aggregate=True)
        torch.cuda.synchronize()
        ev0 = torch.cuda.Event(enable_timing=True); ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record()
        for _ in range(10): e.query(Q3, N=15, aggregate=True)
        ev1.record(); torch.cuda.synchronize()
        ms = ev0.elapsed_time(ev1) / 10
        e.set_option("time_kernels", 1)
        for _ in range(5): e.query(Q3, N=15, aggregate=True)
        torch.cuda.synchronize()
        t = {k: e.stat(f"time_{k}_ns") / 5 / 1e6 for k in ("seed", "scan", "merge", "final")}
        print(f"C3 n_s {ns:2d} K_c {kc:2d}: {ms:.3f} ms/step = {1024 / ms * 1e3:,.0f} queries/s "
              f"(seed {t['seed']:.3f} scan {t['scan']:.3f} merge {t['merge']:.3f} Alg.2 {t['final']:.3f}; "
              f"tc {e.stat('used_tc')}, survivors/pair {e.stat('survivors') / e.stat('pairs'):.1e})", flush=True)
        e.close()
