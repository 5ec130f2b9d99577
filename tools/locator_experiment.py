"""Would a seed that knows where each frame's near matches are pay off at C4?

A "locator" (here plain torch, outside the library) scores every frame against the centroid
of every 32-row block, takes the k best blocks, and computes the exact N-th best distance over
their 32k rows -- an upper bound of the frame's N-th best (N real rows).  The scan is then run
from min(seed, locator) thresholds (tc_debug 64: start from ol_thresholds as they are) and
compared with the library's own seed and with converged thresholds (the limit).  Results must
be identical to the normal query's.
  python tools/locator_experiment.py [rows]"""
import os, sys, time, torch
import numpy as np
sys.path.insert(0, '.')
import synthgen, paper_2006_08861_b200 as ol

torch.backends.cuda.matmul.allow_tf32 = False
spec = synthgen.CONFIGS["C4"].spec
n = int(sys.argv[1]) if len(sys.argv) > 1 else spec.n_entries
n -= n % 32
N = 15
dev = torch.device("cuda", 0)
F, C = synthgen.db_device(spec, 0, n, dev)
NQ = int(os.environ.get("NQ", 1024))
Q, _ = synthgen.render_device(spec, synthgen.query_points(spec, 4242, NQ), dev)
e = ol.Engine(0)
e.upload(F, C, [n], spec.grid())
del C
Q3 = Q.view(-1, 1, 64)


def timed(dbg, tau=None, reps=5):
    tot = {"seed": 0.0, "scan": 0.0}
    surv = 0.0
    for _ in range(reps):
        if tau is not None:
            e.set_option("tc_debug", 0)
            e.query(Q3, N=N)
            e.thresholds().copy_(tau)
        e.set_option("tc_debug", dbg)
        e.set_option("time_kernels", 1)
        e.query(Q3, N=N)
        torch.cuda.synchronize()
        for k in tot: tot[k] += e.stat(f"time_{k}_ns") / 1e6 / reps
        for k in ("merge", "final"): e.stat(f"time_{k}_ns")
        e.set_option("time_kernels", 0)
        surv += e.stat("survivors") / reps
    e.set_option("tc_debug", 0)
    return tot, surv / e.stat("pairs"), e.topk().copy()


for _ in range(2): e.query(Q3, N=N)
t0, s0, ref = timed(0)
print(f"own seed        seed {t0['seed']:.3f} scan {t0['scan']:.3f} ms  survivors/pair {s0:.2e}", flush=True)
tau_final = e.thresholds().clone()
e.set_option("tc_debug", 512); e.query(Q3, N=N); torch.cuda.synchronize()
tau_seed = e.thresholds().clone()
e.set_option("tc_debug", 0)

# the locator: centroid distances (all 64 dims, or the 32-dim prefix), k best blocks per frame
nb = n // 32
Fv = F.view(nb, 32, 64)
for dims in (64, 32):
    cen = torch.empty(nb, dims, device=dev)
    for b in range(0, nb, 1 << 20):
        cen[b:b + (1 << 20)] = Fv[b:b + (1 << 20), :, :dims].mean(1)
    cn = (cen * cen).sum(1)
    torch.cuda.synchronize(); tl = time.perf_counter()
    best_v = torch.full((NQ, 0), 0.0, device=dev); best_i = torch.zeros((NQ, 0), dtype=torch.long, device=dev)
    K = 8
    for b in range(0, nb, 1 << 20):
        d = cn[b:b + (1 << 20)][None, :] - 2.0 * (Q[:, :dims] @ cen[b:b + (1 << 20)].T)
        v, i = torch.topk(d, K, dim=1, largest=False)
        best_v = torch.cat([best_v, v], 1); best_i = torch.cat([best_i, i + b], 1)
        v, j = torch.topk(best_v, K, dim=1, largest=False)
        best_v, best_i = v, torch.gather(best_i, 1, j)
    torch.cuda.synchronize(); tl = time.perf_counter() - tl
    for k in (1, 2, 4, 8):
        rows = (best_i[:, :k, None] * 32 + torch.arange(32, device=dev)).reshape(NQ, -1)
        X = F[rows].double()                                   # [NQ, 32k, 64]
        d2 = ((X - Q.double()[:, None, :]) ** 2).sum(2)
        nth = torch.sort(d2, 1).values[:, N - 1]
        tau_loc = (nth * (1 + 2e-5) + 1e-30).float()
        tau_loc_i = tau_loc.view(torch.int32)
        tau = torch.minimum(tau_seed, tau_loc_i)
        fin = tau_final.view(torch.float32).double()
        ratio = (tau.view(torch.float32).double() / fin.clamp_min(1e-30)).cpu().numpy()
        t1, s1, got = timed(64, tau)
        same = np.array_equal(got, ref)
        print(f"locator dims {dims} k {k} (torch {tl * 1e3:.1f} ms): tau/final median {np.median(ratio):.3f} "
              f"p90 {np.percentile(ratio, 90):.3f} within 1% {np.mean(ratio < 1.01):.2f} | "
              f"scan {t1['scan']:.3f} ms survivors/pair {s1:.2e} identical {same}", flush=True)
t2, s2, got = timed(64, tau_final)
print(f"converged       scan {t2['scan']:.3f} ms  survivors/pair {s2:.2e} identical {np.array_equal(got, ref)}")
ratio = (tau_seed.view(torch.float32).double() / tau_final.view(torch.float32).double().clamp_min(1e-30)).cpu().numpy()
print(f"seed tau/final median {np.median(ratio):.3f} p90 {np.percentile(ratio, 90):.3f}")
