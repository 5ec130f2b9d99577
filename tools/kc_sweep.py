"""C3 (1M rows, 1,024 frames): the CUDA-core scan's coarse prefix K_c (SURVEY §8d sweep
{0 = one-pass, 8, 16, 32}) -- scan time, survivors, fraction of the FP32-issue ceiling --
next to the tensor-core filter."""
import sys, torch
sys.path.insert(0, '.')
import synthgen, paper_2006_08861_b200 as ol
cfg = synthgen.CONFIGS["C3"]; spec = cfg.spec
dev = torch.device("cuda", 0)
F, C = synthgen.db_device(spec, 0, spec.n_entries, dev)
Q, _ = synthgen.render_device(spec, synthgen.query_points(spec, 4242, 1024), dev)
Q3 = Q.view(-1, 1, 64)
pairs = 1024 * spec.n_entries
for kc, tc in [(64, 0), (8, 0), (16, 0), (32, 0), (16, 1)]:
    e = ol.Engine(0, coarse_k=kc)
    e.set_option("tc", tc)
    e.upload(F, C, [spec.n_entries], spec.grid())
    for _ in range(2): e.query(Q3, N=15)
    torch.cuda.synchronize()
    e.set_option("time_kernels", 1)
    for _ in range(5): e.query(Q3, N=15)
    torch.cuda.synchronize()
    t = {k: e.stat(f"time_{k}_ns") / 5 / 1e6 for k in ("seed", "scan", "merge", "final")}
    alu = pairs * 2 * kc / (t["scan"] * 1e-3) / (148 * 128 * 1.965e9)
    print(f"C3 K_c={'one-pass' if kc == 64 else kc} tc={tc} scan {t['scan']:.3f} ms seed {t['seed']:.3f} ms "
          f"survivors/pair {e.stat('survivors') / e.stat('pairs'):.2e}" + ("" if tc else f" FP32-issue frac {alu:.2f}"))
