"""C1 latency of the single-kernel path: per-query device time (CUDA events, graph replay off)
with Algorithm 2 on / off, and the launch sequence (option micro = 0) for comparison."""
import sys, torch
sys.path.insert(0, '.')
import numpy as np
import synthgen, paper_2006_08861_b200 as ol
cfg = synthgen.CONFIGS["C1"]
F, C = synthgen.db_host(cfg.spec)
Q = synthgen.render_host(cfg.spec, synthgen.query_points(cfg.spec, 11, 1))["desc"]
qd = torch.from_numpy(Q[:, None, :].copy()).cuda()
e = ol.Engine(0)
e.upload(F, C, cfg.subspace_sizes, cfg.spec.grid())
for micro in (1, 0):
    e.set_option("micro", micro)
    for agg in (True, False):
        for _ in range(50): e.query(qd, N=cfg.N, aggregate=agg)
        torch.cuda.synchronize()
        s0 = torch.cuda.Event(enable_timing=True); s1 = torch.cuda.Event(enable_timing=True)
        s0.record()
        for _ in range(500): e.query(qd, N=cfg.N, aggregate=agg)
        s1.record(); torch.cuda.synchronize()
        print(f"micro={micro} aggregate={agg}: {s0.elapsed_time(s1) / 500 * 1e3:.1f} us/query, {e.stat('kernels')} launches")

e.set_option("micro", 1)
e.set_option("tc_debug", 32)
e.query(qd, N=cfg.N, aggregate=True)
torch.cuda.synchronize()
print("micro phases (cycles): scan", e.stat("prof0"), "top-N + rows", e.stat("prof1"), "bundle count", e.stat("prof2"),
      "Alg. 2", e.stat("prof3"))
print("  of top-N + rows: own select", e.stat("prof4"), "cluster barrier", e.stat("prof5"), "gather + barrier", e.stat("prof6"),
      "rows", e.stat("prof7"))
