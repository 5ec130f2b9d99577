"""Inline exact re-scoring (option inline_rescore) vs the two exact warps: C2 (20k rows,
1,000 bundles of M = 5), C3 (1M rows, 1,024 frames) and a 12.5M-row C4 shard."""
import sys, torch
sys.path.insert(0, '.')
import synthgen, paper_2006_08861_b200 as ol


def timed(e, Q, agg, reps=10):
    for _ in range(3): e.query(Q, N=15, aggregate=agg)
    torch.cuda.synchronize()
    e.set_option("time_kernels", 1)
    for _ in range(reps): e.query(Q, N=15, aggregate=agg)
    torch.cuda.synchronize()
    t = {k: e.stat(f"time_{k}_ns") / reps / 1e6 for k in ("seed", "scan", "merge", "final")}
    e.set_option("time_kernels", 0)
    return t


cfg = synthgen.CONFIGS["C2"]; spec = cfg.spec
F, C = synthgen.db_host(spec)
video = synthgen.render_host(spec, synthgen.query_points(spec, 5, 1000, "path", 0, 2))["desc"]
firsts = [ol.select_window(1000, m, 5)[0] for m in range(1000)]
Qd = torch.from_numpy(synthgen.gather_windows(video, firsts, 5)).cuda()
e = ol.Engine(0)
e.upload(F, C, cfg.subspace_sizes, spec.grid())
for rep in range(2):
    for v in (0, 1):
        e.set_option("inline_rescore", v)
        t = timed(e, Qd, True)
        print(f"C2 inline {v}: scan {t['scan']:.3f} ms (chunk {e.stat('chunk')}, items {e.stat('items')})", flush=True)
e.close()
c4 = synthgen.CONFIGS["C4"].spec
dev = torch.device("cuda", 0)
for n in (1_000_000, 12_500_000):
    F, C = synthgen.db_device(c4, 0, n, dev)
    e = ol.Engine(0)
    e.upload(F, C, [n], c4.grid())
    del F, C
    Q, _ = synthgen.render_device(c4, synthgen.query_points(c4, 4242, 1024), dev)
    Q3 = Q.view(-1, 1, 64)
    for rep in range(2):
        for v in (0, 1):
            e.set_option("inline_rescore", v)
            t = timed(e, Q3, False, 5)
            print(f"rows {n:,} inline {v}: scan {t['scan']:.3f} ms (chunk {e.stat('chunk')}, items {e.stat('items')})", flush=True)
    e.close()
    torch.cuda.empty_cache()
