"""C3 (1M rows, 1,024 frames): tensor-core filter vs CUDA-core scan, survivors and time."""
import sys, torch
sys.path.insert(0, '.')
import synthgen, paper_2006_08861_b200 as ol
cfgn = sys.argv[1] if len(sys.argv) > 1 else "C3"
cfg = synthgen.CONFIGS[cfgn]; spec = cfg.spec
dev = torch.device("cuda", 0)
F, C = synthgen.db_device(spec, 0, spec.n_entries, dev)
Q, _ = synthgen.render_device(spec, synthgen.query_points(spec, 4242, 1024), dev)
Q3 = Q.view(-1, 1, 64)
for tc, extra in [(1, {}), (0, {}), (1, {"tc_k": 32})]:
    e = ol.Engine(0)
    e.set_option("tc", tc)
    for k, v in extra.items(): e.set_option(k, v)
    e.upload(F, C, [spec.n_entries], spec.grid())
    for _ in range(2): e.query(Q3, N=15)
    torch.cuda.synchronize()
    e.set_option("time_kernels", 1)
    for _ in range(5): e.query(Q3, N=15)
    torch.cuda.synchronize()
    t = {k: e.stat(f"time_{k}_ns") / 5 / 1e6 for k in ("seed", "scan", "merge", "final")}
    print(f"{cfgn} tc={tc} {extra} used_tc={e.stat('used_tc')} seed {t['seed']:.3f} scan {t['scan']:.3f} ms survivors/pair {e.stat('survivors')/e.stat('pairs'):.2e}")
