"""How much of the C4 scan is start-up survivors?  Times the scan seeded as usual, then
seeded with the converged thresholds of the previous query (tc_debug 64: start from
ol_thresholds as they are), which is the limit any better seed could reach.
  python tools/seed_gain.py [rows]"""
import os, sys, torch
sys.path.insert(0, '.')
import synthgen, paper_2006_08861_b200 as ol
spec = synthgen.CONFIGS["C4"].spec
n = int(sys.argv[1]) if len(sys.argv) > 1 else spec.n_entries
dev = torch.device("cuda", 0)
F, C = synthgen.db_device(spec, 0, n, dev)
NQ = int(os.environ.get("NQ", 1024))
Q, _ = synthgen.render_device(spec, synthgen.query_points(spec, 4242, NQ), dev)
e = ol.Engine(0)
e.upload(F, C, [n], spec.grid())
del F, C
Q3 = Q.view(-1, 1, 64)


def run(dbg, reps=5, extra=None):
    tot = {"seed": 0.0, "scan": 0.0}
    surv = flag = 0
    for _ in range(reps):
        e.set_option("tc_debug", 0)
        e.query(Q3, N=15)                     # converged thresholds left in ol_thresholds
        e.set_option("tc_debug", dbg)
        if extra: extra()
        e.set_option("time_kernels", 1)
        e.query(Q3, N=15)
        torch.cuda.synchronize()
        for k in tot: tot[k] += e.stat(f"time_{k}_ns") / 1e6 / reps
        for k in ("merge", "final"): e.stat(f"time_{k}_ns")
        e.set_option("time_kernels", 0)
        surv += e.stat("survivors") / reps
        flag += e.stat("flagged") / reps
    return tot, surv / e.stat("pairs"), flag


for _ in range(2): e.query(Q3, N=15)
for name, dbg in (("own seed", 0), ("converged (tc_debug 64)", 64)):
    t, s, f = run(dbg)
    print(f"{name:26s} seed {t['seed']:.3f} scan {t['scan']:.3f} ms  survivors/pair {s:.2e}  flagged events {f:.0f}", flush=True)
