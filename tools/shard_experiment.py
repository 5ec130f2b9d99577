"""Per-rank cost of C4 sharded over W GPUs, measured on ONE GPU (one gpurun call has one):
every rank's shard is built in turn, its seed thresholds are taken (tc_debug 512 stops
ol_query after the seed), their minimum over ranks is what the in-library NCCL path's
MIN all-reduce hands every rank.  Then rank r's full query is timed with (a) its own
seed and (b) the shared minimum (tc_debug 64: start from the values in ol_thresholds),
for the automatic filter shape and the alternatives given in CONFIGS.

  python tools/shard_experiment.py W [ranks] [configs]   e.g. 8 0,7 auto,k32,k64p0
"""
import sys
import time

import torch

sys.path.insert(0, ".")
import synthgen
import paper_2006_08861_b200 as ol

W = int(sys.argv[1]) if len(sys.argv) > 1 else 8
RANKS = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "0").split(",")]
CONFIGS = (sys.argv[3] if len(sys.argv) > 3 else "auto").split(",")
spec = synthgen.CONFIGS["C4"].spec
n = spec.n_entries
dev = torch.device("cuda", 0)
Q, _ = synthgen.render_device(spec, synthgen.query_points(spec, 4242, 1024), dev)
Q3 = Q.view(1024, 1, 64)


def opts(e, cfg):
    e.set_option("tc_k", 0); e.set_option("pair", 1)
    if "k32" in cfg: e.set_option("tc_k", 32)
    if "k64" in cfg: e.set_option("tc_k", 64)
    if "p0" in cfg: e.set_option("pair", 0)
    if "p2" in cfg: e.set_option("pair", 2)


t0 = time.time()
seeds = []
for r in range(W):
    b, c = ol.shard_range(n, r, W)
    F, C = synthgen.db_device(spec, b, c, dev)
    e = ol.Engine(0, rank=r, world=W, exchange="torch")
    e.upload(F, C, [n], spec.grid())
    del F, C
    e.set_option("tc_debug", 512)
    e.query(Q3, N=15, aggregate=True, exchange=False)
    seeds.append(e.thresholds().clone())
    e.close()
    torch.cuda.empty_cache()
shared = torch.stack(seeds).min(dim=0).values
own_mean = torch.stack([s.view(torch.float32) for s in seeds]).mean().item()
print(f"W={W}: seeds of {W} ranks in {time.time() - t0:.1f} s; mean own seed tau {own_mean:.5f}, "
      f"shared {shared.view(torch.float32).mean().item():.5f}", flush=True)

for r in RANKS:
    b, c = ol.shard_range(n, r, W)
    F, C = synthgen.db_device(spec, b, c, dev)
    for cfg in CONFIGS:
        e = ol.Engine(0, rank=r, world=W, exchange="torch")
        opts(e, cfg)
        e.upload(F, C, [n], spec.grid())
        for mode in ("own", "shared"):
            for _ in range(2):
                e.set_option("tc_debug", 0)
                e.query(Q3, N=15, aggregate=True, exchange=False)
            torch.cuda.synchronize()
            reps = 5
            tot = {"seed": 0.0, "scan": 0.0, "merge": 0.0}
            surv = 0
            for _ in range(reps):
                if mode == "shared":
                    e.set_option("tc_debug", 0)
                    e.set_option("tc_debug", 512)
                    e.query(Q3, N=15, aggregate=True, exchange=False)         # this shape's buffers + own seed
                    e.thresholds().copy_(shared)
                    e.set_option("tc_debug", 64)
                else:
                    e.set_option("tc_debug", 0)
                e.set_option("time_kernels", 1)
                e.query(Q3, N=15, aggregate=True, exchange=False)
                torch.cuda.synchronize()
                for k in tot:
                    tot[k] += e.stat(f"time_{k}_ns") / 1e6
                e.stat("time_final_ns")
                e.set_option("time_kernels", 0)
                surv += e.stat("survivors")
            t = {k: v / reps for k, v in tot.items()}
            if mode == "shared":   # the shared run's seed is the own seed + the all-reduce (not timed here)
                t["seed"] = own_seed
            else:
                own_seed = t["seed"]
            print(f"rank {r}/{W} rows {c:,} cfg {cfg} tc_k {e.stat('tc_k')} pair {e.stat('used_pair')} "
                  f"{mode:6s}: seed {t['seed']:.3f} scan {t['scan']:.3f} merge {t['merge']:.3f} ms, "
                  f"survivors {surv / reps / (1024 * c):.3e}", flush=True)
        e.close()
    del F, C
    torch.cuda.empty_cache()

# ---- in-scan threshold sharing (NCCL mode's peer-memory MINs), emulated: all W shards'
# queries in flight at once on one GPU, linked by ol_tau_share_emulate (argv[4] == "share")
if len(sys.argv) > 4 and sys.argv[4] == "share":
    engines, streams = [], []
    for r in range(W):
        b, c = ol.shard_range(n, r, W)
        F, C = synthgen.db_device(spec, b, c, dev)
        st = torch.cuda.Stream()
        e = ol.Engine(0, rank=r, world=W, exchange="torch", stream=st)
        e.upload(F, C, [n], spec.grid())
        del F, C
        engines.append(e); streams.append(st)
    torch.cuda.synchronize()
    for e in engines:
        e.query(Q3, N=15, aggregate=True, exchange=False)
    torch.cuda.synchronize()
    for linked in (False, True):
        if linked:
            ol.tau_share_emulate(engines)
        for rep in range(2):
            for e in engines:   # own seeds, then the shared minimum (what the NCCL MIN all-reduce gives)
                e.set_option("tc_debug", 512)
                e.query(Q3, N=15, aggregate=True, exchange=False)
            torch.cuda.synchronize()
            shared = torch.stack([e.thresholds().clone() for e in engines]).min(dim=0).values
            for e in engines:
                e.thresholds().copy_(shared)
                e.set_option("tc_debug", 64)
            torch.cuda.synchronize()
            t0 = time.time()
            for e in engines:
                e.query(Q3, N=15, aggregate=True, exchange=False)
            torch.cuda.synchronize()
            wall = (time.time() - t0) * 1e3
        surv = [e.stat("survivors") / (1024 * ol.shard_range(n, r, W)[1]) for r, e in enumerate(engines)]
        print(f"W={W} concurrent on one GPU, tau sharing {'ON ' if linked else 'off'}: survivors per rank "
              f"mean {sum(surv) / W:.3e} (min {min(surv):.3e}, max {max(surv):.3e}); all W scans {wall:.1f} ms wall",
              flush=True)
