"""Seed select A/B (option seed_select 0 = warp gather where it applies, 1 = CTA / radix;
the 8,192-sample measurement in DESIGN used a build routing <= 8,192 samples to the warp):
seed time at C4-shaped DBs (argv[1] rows, 1,024 frames, one subspace) and C3 split into
5 / 50 subspaces."""
import sys, torch
sys.path.insert(0, '.')
import synthgen, paper_2006_08861_b200 as ol
dev = torch.device("cuda", 0)


def seed_ms(e, Q3, sel, reps=10):
    e.set_option("seed_select", sel)
    for _ in range(3): e.query(Q3, N=15)
    torch.cuda.synchronize()
    e.set_option("time_kernels", 1)
    for _ in range(reps): e.query(Q3, N=15)
    torch.cuda.synchronize()
    t = {k: e.stat(f"time_{k}_ns") / reps / 1e6 for k in ("seed", "scan", "merge", "final")}
    e.set_option("time_kernels", 0)
    return t


for name, n, nss in (("C4", int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000, (1,)), ("C3", 1_000_000, (1, 5, 50))):
    spec = synthgen.CONFIGS[name].spec
    F, C = synthgen.db_device(spec, 0, n, dev)
    Q, _ = synthgen.render_device(spec, synthgen.query_points(spec, 4242, 1024), dev)
    Q3 = Q.view(-1, 1, 64)
    for ns in nss:
        sizes = [n // ns + (1 if i < n % ns else 0) for i in range(ns)]
        e = ol.Engine(0)
        e.upload(F, C, sizes, spec.grid())
        for rep in range(2):
            for sel in (0, 1):
                t = seed_ms(e, Q3, sel)
                print(f"{name} rows {n:,} n_s {ns} seed_select {sel}: seed {t['seed']:.3f} scan {t['scan']:.3f} ms", flush=True)
        e.close()
    del F, C
