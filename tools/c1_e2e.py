"""C1 end to end through the public API (pinned host frames in, candidates + estimates out):
where the microseconds go -- the device time of the query alone, and the host wall time of
ol_query (+H2D), ol_get_topk and ol_get_estimates (each D2H + stream sync) per step."""
import sys, time, torch
sys.path.insert(0, '.')
import numpy as np
import synthgen, paper_2006_08861_b200 as ol
cfg = synthgen.CONFIGS["C1"]
F, C = synthgen.db_host(cfg.spec)
Q = synthgen.render_host(cfg.spec, synthgen.query_points(cfg.spec, 11, 1))["desc"]
e = ol.Engine(0)
e.upload(F, C, cfg.subspace_sizes, cfg.spec.grid())
Qh = torch.from_numpy(Q[:, None, :].copy()).pin_memory()
Qn = Qh.numpy()
e.query(Qn, N=cfg.N, aggregate=True)
nc = e.candidate_count()
res = torch.empty(nc * 32, dtype=torch.uint8).pin_memory()
est = torch.empty(ol.ESTIMATE_DTYPE.itemsize, dtype=torch.uint8).pin_memory()
for _ in range(200):
    e.query(Qn, N=cfg.N, aggregate=True); e.topk_into(res); e.estimates_into(est)
torch.cuda.synchronize()
n = 2000
tq = tt = te = 0.0
t0 = time.perf_counter()
for _ in range(n):
    a = time.perf_counter(); e.query(Qn, N=cfg.N, aggregate=True)
    b = time.perf_counter(); e.topk_into(res)
    c = time.perf_counter(); e.estimates_into(est)
    d = time.perf_counter()
    tq += b - a; tt += c - b; te += d - c
wall = (time.perf_counter() - t0) / n * 1e6
print(f"C1 e2e: {wall:.1f} us per step = query {tq / n * 1e6:.1f} + topk {tt / n * 1e6:.1f} + estimates {te / n * 1e6:.1f} us (host wall)")
t0 = time.perf_counter()
for _ in range(n):
    e.query(Qn, N=cfg.N, aggregate=True); e.results_into(res, est)
print(f"C1 e2e with one fetch (ol_get_results): {(time.perf_counter() - t0) / n * 1e6:.1f} us per step")
