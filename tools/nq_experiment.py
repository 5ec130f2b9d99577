"""Scan time vs query frames (C4 database): tensor-core filter vs CUDA-core scan."""
import sys, torch
sys.path.insert(0, '.')
import synthgen, paper_2006_08861_b200 as ol
spec = synthgen.CONFIGS["C4"].spec
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
dev = torch.device("cuda", 0)
F, C = synthgen.db_device(spec, 0, n, dev)
Q, _ = synthgen.render_device(spec, synthgen.query_points(spec, 4242, 1024), dev)
e = ol.Engine(0)
e.upload(F, C, [n], spec.grid())
import os
if os.environ.get("SEEDS"): e.set_option("seed_samples", int(os.environ["SEEDS"]))
for nq in [int(x) for x in sys.argv[2].split(',')]:
    Q3 = Q[:nq].contiguous().view(-1, 1, 64)
    for tc, pair, sk in [(1, 1, 1), (0, 1, 1)][:int(os.environ.get("ARMS", 2))]:
        e.set_option("tc", tc); e.set_option("pair", pair); e.set_option("seed_kernel", sk)
        for _ in range(2): e.query(Q3, N=15)
        torch.cuda.synchronize()
        e.set_option("time_kernels", 1)
        for _ in range(5): e.query(Q3, N=15)
        torch.cuda.synchronize()
        t = {k: e.stat(f"time_{k}_ns") / 5 / 1e6 for k in ("seed", "scan", "merge", "final")}
        e.set_option("time_kernels", 0)
        print(f"nq={nq} tc={tc} used_tc={e.stat('used_tc')} pair={e.stat('used_pair')} tc_k={e.stat('tc_k')} seed {t['seed']:.3f} scan {t['scan']:.3f} total {sum(t.values()):.3f} ms")
