"""C2 (20k rows, 5 subspaces, 1,000 bundles of M = 5, Alg. 2): stage times with the warp
seed select (seed_select 0) and the radix warp select (1)."""
import sys, torch
sys.path.insert(0, '.')
import synthgen, paper_2006_08861_b200 as ol
cfg = synthgen.CONFIGS["C2"]; spec = cfg.spec
F, C = synthgen.db_host(spec)
video = synthgen.render_host(spec, synthgen.query_points(spec, 5, 1000, "path", 0, 2))["desc"]
firsts = [ol.select_window(1000, m, 5)[0] for m in range(1000)]
Qd = torch.from_numpy(synthgen.gather_windows(video, firsts, 5)).cuda()
e = ol.Engine(0)
e.upload(F, C, cfg.subspace_sizes, spec.grid())
for rep in range(2):
    for sel in (0, 1):
        e.set_option("seed_select", sel)
        for _ in range(3): e.query(Qd, N=15, aggregate=True)
        torch.cuda.synchronize()
        e.set_option("time_kernels", 1)
        for _ in range(10): e.query(Qd, N=15, aggregate=True)
        torch.cuda.synchronize()
        t = {k: e.stat(f"time_{k}_ns") / 10 / 1e6 for k in ("seed", "scan", "merge", "final")}
        e.set_option("time_kernels", 0)
        print(f"C2 seed_select {sel}: " + " ".join(f"{k} {v:.3f}" for k, v in t.items())
              + f" ms, sum {sum(t.values()):.3f} -> {1000 / sum(t.values()) * 1e3:,.0f} localisations/s", flush=True)
