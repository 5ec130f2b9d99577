"""C1 (2,000 rows, 1 frame, N = 5): per-query latency with and without the tau seed."""
import sys, torch
sys.path.insert(0, '.')
import synthgen, paper_2006_08861_b200 as ol
cfg = synthgen.CONFIGS["C1"]; spec = cfg.spec
F, C = synthgen.db_host(spec)
Q = synthgen.render_host(spec, synthgen.query_points(spec, 5, 1))["desc"][:, None, :]
Qd = torch.from_numpy(Q).cuda()
for opts in ({}, {"tau_seed": 0}):
    e = ol.Engine(0)
    for k, v in opts.items(): e.set_option(k, v)
    e.upload(F, C, cfg.subspace_sizes, spec.grid())
    for _ in range(20): e.query(Qd, N=cfg.N, aggregate=True)
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True); ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(200): e.query(Qd, N=cfg.N, aggregate=True)
    ev1.record(); torch.cuda.synchronize()
    print(f"C1 {opts}: {ev0.elapsed_time(ev1) / 200 * 1e3:.1f} us/query, kernels {e.stat('kernels')}")
