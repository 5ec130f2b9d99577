"""C2 (20k rows in 5 path subspaces, 1,000 bundles of M = 5, Alg. 2): scan paths and coarse widths (tc auto vs CUDA-core kc 0 / 8 / 32, qtile 32)."""
import sys, torch
sys.path.insert(0, '.')
import synthgen, paper_2006_08861_b200 as ol
cfg = synthgen.CONFIGS["C2"]; spec = cfg.spec
F, C = synthgen.db_host(spec)
video = synthgen.render_host(spec, synthgen.query_points(spec, 5, 1000, "path", 0, 2))["desc"]
firsts = [ol.select_window(1000, m, 5)[0] for m in range(1000)]
Q = synthgen.gather_windows(video, firsts, 5)
Qd = torch.from_numpy(Q).cuda()
for kc, tc, opts in [(16, -1, {}), (0, 0, {}), (0, 0, {"qtile": 32}), (8, 0, {}), (32, 0, {})]:
    e = ol.Engine(0, coarse_k=kc); e.set_option("tc", tc)
    for k, v in opts.items(): e.set_option(k, v)
    e.upload(F, C, cfg.subspace_sizes, spec.grid())
    for _ in range(3): e.query(Qd, N=15, aggregate=True)
    torch.cuda.synchronize()
    e.set_option("time_kernels", 1)
    ev0 = torch.cuda.Event(enable_timing=True); ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(10): e.query(Qd, N=15, aggregate=True)
    ev1.record(); torch.cuda.synchronize()
    t = {k: round(e.stat(f"time_{k}_ns") / 10 / 1e6, 3) for k in ("seed", "scan", "merge", "final")}
    ms = ev0.elapsed_time(ev1) / 10
    print(f"C2 kc={kc} tc={tc} {opts} survivors {e.stat('survivors')/e.stat('pairs'):.2e} {ms:.3f} ms -> {1000/ms*1e3:.0f} loc/s {t}")
