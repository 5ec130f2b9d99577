"""C3 with n_s = 5 / 50 subspaces: seed sample count vs seed + scan time (env INLINE: the
inline_rescore option)."""
import sys, torch
sys.path.insert(0, '.')
import synthgen, paper_2006_08861_b200 as ol
cfg = synthgen.CONFIGS["C3"]; spec = cfg.spec
n = spec.n_entries
dev = torch.device("cuda", 0)
F, C = synthgen.db_device(spec, 0, n, dev)
Q, _ = synthgen.render_device(spec, synthgen.query_points(spec, 4242, 1024), dev)
Q3 = Q.view(-1, 1, 64)
for ns in (5, 50):
    sizes = [n // ns + (1 if i < n % ns else 0) for i in range(ns)]
    e = ol.Engine(0, coarse_k=16)
    import os
    if os.environ.get("INLINE"): e.set_option("inline_rescore", int(os.environ["INLINE"]))
    e.upload(F, C, sizes, spec.grid())
    for S in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "0,128,256,512,1024,2048").split(",")]:
        e.set_option("seed_samples", S) if S else e.set_option("seed_samples", 0)
        if S and S < 16: continue
        for _ in range(3): e.query(Q3, N=15, aggregate=True)
        torch.cuda.synchronize()
        e.set_option("time_kernels", 1)
        for _ in range(5): e.query(Q3, N=15, aggregate=True)
        torch.cuda.synchronize()
        t = {k: e.stat(f"time_{k}_ns") / 5 / 1e6 for k in ("seed", "scan", "merge", "final")}
        e.set_option("time_kernels", 0)
        print(f"n_s {ns} samples {S or 'auto'}: seed {t['seed']:.3f} scan {t['scan']:.3f} sum {t['seed'] + t['scan']:.3f} survivors {e.stat('survivors') / e.stat('pairs'):.1e}", flush=True)
    e.close()
