"""Per-role cycle counters of the tensor-core scan (tc_debug 32), per 256-row tile, at a
C4-shaped DB of argv[1] rows: with the library's own seed and from converged thresholds
(tc_debug 32|64), so the steady-state pipeline can be told apart from the start-up survivors.
  python tools/tc_roles.py [rows]"""
import os, sys, torch
sys.path.insert(0, '.')
import synthgen, paper_2006_08861_b200 as ol
spec = synthgen.CONFIGS["C4"].spec
n = int(sys.argv[1]) if len(sys.argv) > 1 else spec.n_entries
dev = torch.device("cuda", 0)
F, C = synthgen.db_device(spec, 0, n, dev)
Q, _ = synthgen.render_device(spec, synthgen.query_points(spec, 4242, 1024), dev)
e = ol.Engine(0)
e.upload(F, C, [n], spec.grid())
del F, C
Q3 = Q.view(-1, 1, 64)
for _ in range(2): e.query(Q3, N=15)
for name, dbg in (("own seed", 32), ("converged", 32 | 64)):
    e.set_option("tc_debug", 0); e.query(Q3, N=15)
    e.set_option("tc_debug", dbg); e.set_option("time_kernels", 1)
    for i in range(32): e.stat(f"prof{i}")
    e.query(Q3, N=15); torch.cuda.synchronize()
    ms = e.stat("time_scan_ns") / 1e6
    for k in ("seed", "merge", "final"): e.stat(f"time_{k}_ns")
    e.set_option("time_kernels", 0)
    P = [e.stat(f"prof{i}") for i in range(32)]
    T = max(P[9], 1)                 # tile passes, all CTAs
    W = T * 8                        # epilogue warp-tiles (16 warps, alternate tiles)
    print(f"{name}: scan {ms:.3f} ms, CTA cycles/tile {P[8] / T:.0f}; MMA per tile: wait-full {P[0] / T:.0f} "
          f"wait-tempty {P[1] / T:.0f} issue {P[16] / T:.0f} commit {P[18] / T:.0f} tma-lat {P[17] / T:.0f}; "
          f"epilogue per warp-tile: wait-tfull {P[6] / W:.0f} ld {P[12] / W:.0f} math {P[13] / W:.0f} "
          f"tile {P[11] / W:.0f}; events {P[4]} cold-cycles {P[2]}; exact busy {P[7] / max(P[8], 1):.2f} of CTA life",
          flush=True)
e.set_option("tc_debug", 0)
