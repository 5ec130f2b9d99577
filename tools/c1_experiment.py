"""C1 (2,000 rows, 1 frame, N = 5): per-query device latency with and without the tau
seed, eager and with CUDA-graph replay (option "graph")."""
import sys, torch
sys.path.insert(0, '.')
import synthgen, paper_2006_08861_b200 as ol
cfg = synthgen.CONFIGS["C1"]; spec = cfg.spec
F, C = synthgen.db_host(spec)
Q = synthgen.render_host(spec, synthgen.query_points(spec, 5, 1))["desc"][:, None, :]
Qd = torch.from_numpy(Q).cuda()
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for opts in ({}, {"graph": 1}, {"graph": 1, "tau_seed": 0}, {"graph": 1, "chunk": 512},
                 {"graph": 1, "chunk": 256}, {"graph": 1, "chunk": 128}, {"graph": 1, "chunk": 64},
                 {"graph": 1, "chunk": 256, "seed_samples": 64}, {"graph": 1, "chunk": 128, "qtile": 8}):
        e = ol.Engine(0)
        for k, v in opts.items(): e.set_option(k, v)
        e.upload(F, C, cfg.subspace_sizes, spec.grid())
        for _ in range(20): e.query(Qd, N=cfg.N, aggregate=True)
        ref = e.topk()
        torch.cuda.synchronize()
        ev0 = torch.cuda.Event(enable_timing=True); ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record(s)
        for _ in range(500): e.query(Qd, N=cfg.N, aggregate=True)
        ev1.record(s); torch.cuda.synchronize()
        print(f"C1 {opts}: {ev0.elapsed_time(ev1) / 500 * 1e3:.1f} us/query, kernels {e.stat('kernels')}, "
              f"replays {e.stat('graph_replays')}", flush=True)
