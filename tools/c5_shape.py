"""C5-shaped queries (10M-row DB, 5 frames, N = 15, Alg. 2): per-stage device times for the
automatic path, the CUDA-core scan variants and the tensor-core filter at tc_k 32 / 64
(the plane is chosen at upload: one engine per tc_k)."""
import sys, torch
sys.path.insert(0, '.')
import synthgen, paper_2006_08861_b200 as ol
cfg = synthgen.CONFIGS["C5"]; spec = cfg.spec
n = spec.n_entries
B = int(sys.argv[1]) if len(sys.argv) > 1 else 5
dev = torch.device("cuda", 0)
F, C = synthgen.db_device(spec, 0, n, dev)
Q, _ = synthgen.render_device(spec, synthgen.query_points(spec, 4242, B), dev)
Q3 = Q.view(1, B, 64) if B % 2 else Q.view(B, 1, 64)
for tck, opts in ((0, {}), (0, {"tc": 0, "scan2": 1}), (0, {"tc": 0, "scan2": 2}), (32, {"tc": 1}), (64, {"tc": 1})):
    e = ol.Engine(0)
    if tck: e.set_option("tc_k", tck)
    for k, v in opts.items(): e.set_option(k, v)
    e.upload(F, C, [n], spec.grid())
    for _ in range(3): e.query(Q3, N=cfg.N, aggregate=True)
    torch.cuda.synchronize()
    e.set_option("time_kernels", 1)
    for _ in range(10): e.query(Q3, N=cfg.N, aggregate=True)
    torch.cuda.synchronize()
    t = {k: e.stat(f"time_{k}_ns") / 10 / 1e6 for k in ("seed", "scan", "merge", "final")}
    e.set_option("time_kernels", 0)
    ev0 = torch.cuda.Event(enable_timing=True); ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(20): e.query(Q3, N=cfg.N, aggregate=True)
    ev1.record(); torch.cuda.synchronize()
    print(f"B={B} tc_k={e.stat('tc_k')} {opts} used_tc {e.stat('used_tc')}: step {ev0.elapsed_time(ev1) / 20:.3f} ms; "
          f"seed {t['seed']:.3f} scan {t['scan']:.3f} merge {t['merge']:.3f} final {t['final']:.3f}; "
          f"survivors/pair {e.stat('survivors') / e.stat('pairs'):.2e}", flush=True)
    e.close()
