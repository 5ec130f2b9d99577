"""Small cases for compute-sanitizer (memcheck / racecheck / synccheck / initcheck; one tool
per gpurun call, B200_PROFILING.md): every kernel of the library on the smallest inputs that
reach it, each result still checked against the oracle.

  compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_cases.py [fuzz_cases]

Cases: C1 (CUDA-core scan2 path, seed, merge with candidates, Alg. 2), a 3-bundle M = 3 query
over 2 subspaces (scan_kernel), the tensor-core filter with single CTAs and with CTA pairs
(cta_group::2), the world-2 logical-shard merge (merge_ranks + candidates) and the emulated
peer-memory exchange, standalone Alg. 2 with negative tiles, NEXT-1 shift re-scoring,
descriptor extraction, graph replay, and `fuzz_cases` seeded random cases of tools/fuzz_tc.py
(sizes capped small)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "tools")):
    if p not in sys.path:
        sys.path.insert(0, p)
import oracle  # noqa: E402
import synthgen  # noqa: E402
import paper_2006_08861_b200 as ol  # noqa: E402
from gpu_helpers import assert_candidates_equal, assert_estimates_equal  # noqa: E402


_Engine = ol.Engine


def _engine(*args, **kw):
    """Every engine of these cases poisons its buffers (OL_POISON=1: padding rows / coords NaN
    bytes, per-query outputs garbage-filled before every query) -- the initcheck stand-in."""
    e = _Engine(*args, **kw)
    if os.environ.get("OL_POISON") == "1":
        e.set_option("poison", 1)
    return e


ol.Engine = _engine


def main(n_fuzz: int):
    done = []
    # C1: 2,000 rows, one frame, N = 5 (scan2 + seed + merge + Alg. 2)
    cfg = synthgen.CONFIGS["C1"]
    F, C = synthgen.db_host(cfg.spec)
    Q = synthgen.render_host(cfg.spec, synthgen.query_points(cfg.spec, 11, 1))["desc"][:, None, :]
    e = ol.Engine(0)
    e.upload(F, C, cfg.subspace_sizes, cfg.spec.grid())
    e.query(Q, N=5, aggregate=True)
    ref = oracle.retrieve(cfg.subspace_sizes, F, C, Q, 5)
    assert_candidates_equal(e.topk(), ref, "C1"); assert_estimates_equal(e.estimates(), ref, ctx="C1")
    done.append("C1")
    # graph replay of the same shape (device frames)
    e.set_option("graph", 1)
    qd = torch.from_numpy(np.ascontiguousarray(Q)).cuda()
    for _ in range(2):
        e.query(qd, N=5, aggregate=True)
    assert e.stat("graph_replays") == 1
    assert_candidates_equal(e.topk(), ref, "C1 graph")
    done.append("graph")
    # 2 subspaces, 3 bundles of M = 3 with 40 frames -> scan_kernel (qt > 16)
    spec = synthgen.Spec(seed=3, n_floors=1, paths=2, frames_per_path=1500, path_y0=50.0)
    F, C = synthgen.db_host(spec)
    V = synthgen.render_host(spec, synthgen.query_points(spec, 5, 120))["desc"]
    Qb = np.ascontiguousarray(V[:42].reshape(14, 3, 64))
    e = ol.Engine(0)
    e.upload(F, C, [1500, 1500], spec.grid())
    e.set_option("tc", 0)
    e.query(Qb, N=15, aggregate=True)
    ref = oracle.retrieve([1500, 1500], F, C, Qb, 15)
    assert_candidates_equal(e.topk(), ref, "scan"); assert_estimates_equal(e.estimates(), ref, ctx="scan")
    done.append("scan_kernel")
    # tensor-core filter: single CTAs (tc_k 32 and 64), then CTA pairs over 2 query blocks
    for tck, pair, nq in ((32, 0, 70), (64, 0, 70), (64, 2, 200)):
        e = ol.Engine(0)
        e.set_option("tc", 1); e.set_option("tc_k", tck); e.set_option("pair", pair)
        e.upload(F, C, [1500, 1500], spec.grid())
        Qt = np.ascontiguousarray(V[:nq][:, None, :]) if nq <= len(V) else None
        if Qt is None:
            Vt = synthgen.render_host(spec, synthgen.query_points(spec, 9, nq))["desc"]
            Qt = np.ascontiguousarray(Vt[:, None, :])
        e.query(Qt, N=9, aggregate=False)
        assert e.stat("used_tc") == 1 and e.stat("used_pair") == (1 if pair else 0)
        assert_candidates_equal(e.topk(), oracle.retrieve([1500, 1500], F, C, Qt, 9), f"tc k{tck} pair{pair}")
        done.append(f"tcscan k{tck} pair{pair}")
    # inline exact re-scoring in the epilogue (short work items; per-frame list locks)
    e = ol.Engine(0)
    e.set_option("tc", 1); e.set_option("inline_rescore", 1)
    e.upload(F, C, [1500, 1500], spec.grid())
    Qt = np.ascontiguousarray(V[:70][:, None, :])
    e.query(Qt, N=9, aggregate=True)
    assert e.stat("used_tc") == 1
    ref = oracle.retrieve([1500, 1500], F, C, Qt, 9)
    assert_candidates_equal(e.topk(), ref, "tc inline"); assert_estimates_equal(e.estimates(), ref, ctx="tc inline")
    done.append("tcscan inline")
    # world-2 logical shards: payload + merge_ranks + candidates; and the emulated p2p kernel
    Qs = np.ascontiguousarray(V[:20][:, None, :])
    ref = oracle.retrieve([1500, 1500], F, C, Qs, 7)
    engines, pays = [], []
    for r in range(2):
        es = ol.Engine(0, rank=r, world=2, exchange="torch")
        rows = np.concatenate([np.arange(i * 1500 + b, i * 1500 + b + c) for i in range(2)
                               for b, c in [ol.shard_range(1500, r, 2)]])
        es.upload(F[rows], C[rows], [1500, 1500], spec.grid())
        es.query(Qs, N=7, aggregate=True, exchange=False)
        pays.append(es.payload())
        engines.append(es)
    g = torch.cat(pays)
    for es in engines:
        es.finalize_gathered(g)
        assert_candidates_equal(es.topk(), ref, "shards"); assert_estimates_equal(es.estimates(), ref, ctx="shards")
    for r, es in enumerate(engines):
        es.p2p_open(2, r, 1 << 16)
    for es in engines:
        es.query(Qs, N=7, aggregate=True, exchange=False)
    ol.p2p_emulate(engines)
    for es in engines:
        assert_candidates_equal(es.topk(), ref, "p2p")
    done.append("shards+p2p")
    # NK10 split over a cluster (N > 32: the rounds select), and the merge's gather / fallback
    rng = np.random.default_rng(5)
    Fm = np.abs(rng.standard_normal((5000, 64))).astype(np.float32)
    Fm /= np.linalg.norm(Fm, axis=1, keepdims=True)
    Cm = rng.integers(0, 60, (5000, 2)).astype(np.int32)
    Qm = np.ascontiguousarray((Fm[[7, 4000, 123]] + 1e-3).astype(np.float32).reshape(3, 1, 64))
    for N in (5, 40):
        e = ol.Engine(0)
        e.upload(Fm, Cm, [4990, 10], (64, 64))
        e.query(Qm, N=N, aggregate=True)
        assert e.stat("used_micro") == 1
        ref = oracle.retrieve([4990, 10], Fm, Cm, Qm, N)
        assert_candidates_equal(e.topk(), ref, f"micro N {N}"); assert_estimates_equal(e.estimates(), ref, ctx=f"micro N {N}")
        for scan in (0, 1):
            e = ol.Engine(0)
            e.set_option("micro", 0); e.set_option("chunk", 512); e.set_option("merge_scan", scan)
            e.upload(Fm, Cm, [4990, 10], (64, 64))
            e.query(Qm, N=N, aggregate=True)
            assert_candidates_equal(e.topk(), ref, f"merge N {N} scan {scan}")
    done.append("micro+merge")
    # standalone Alg. 2 with negative tiles
    rng = np.random.default_rng(4)
    xy = rng.integers(-30, 30, (320, 2)).astype(np.int32)
    est = ol.Engine(0).aggregate(xy, np.array([0, 100, 300, 320], np.uint32))   # (the last: one warp)
    for b, (lo, hi) in enumerate(((0, 100), (100, 300), (300, 320))):
        r = oracle.aggregate(xy[lo:hi])
        assert (est[b]["x"], est[b]["y"]) == (r.x, r.y)
    done.append("aggregate")
    # NEXT-1 shift re-scoring and NEXT-3 extraction
    sp = synthgen.Spec(seed=45, n_floors=1, paths=1, frames_per_path=300)
    F1, C1 = synthgen.db_host(sp)
    P1 = synthgen.render_host(sp, synthgen.query_points(sp, 0, 300, "path", 0, 0), profiles=True)["profile"]
    rq = synthgen.render_host(sp, synthgen.query_points(sp, 6, 3), profiles=True)
    e = ol.Engine(0)
    e.upload(F1, C1, [300], sp.grid()); e.upload_profiles(P1.astype(np.float32))
    e.query(rq["desc"][:, None, :], N=3, aggregate=False)
    sh, d2 = e.shift_rescore(rq["profile"].astype(np.float32))
    c = e.topk()
    for i in range(len(c)):
        rd, rs = oracle.shift_distance(rq["profile"][c["bundle"][i]].astype(np.float32), P1[c["frame"][i]].astype(np.float32))
        assert int(sh[i]) == rs and d2[i] == rd
    d32, deg, d64 = e.extract_features(rq["profile"], want64=True)
    for i in range(3):
        cr, dg = oracle.extract_feature(rq["profile"][i])
        assert dg == bool(deg[i]) and np.max(np.abs(d64[i] - cr)) <= 1e-13
    done.append("shift+extract")
    # seeded random cases (small)
    if n_fuzz:
        import fuzz_tc
        fuzz_tc.run(secs=1e9, seed=77, max_cases=n_fuzz)
        done.append(f"fuzz x{n_fuzz}")
    torch.cuda.synchronize()
    e = _Engine(0)
    checked, fail = e.stat("checked"), e.stat("check")
    if checked:
        assert fail == 0, f"device bounds check failed: translation unit {fail >> 24}, line {fail & 0xFFFFFF}"
    print("sanitize cases ok:", ", ".join(done), f"| library {'CHECKED (device bounds checks: 0 failures)' if checked else 'product'}"
          f" | poison {'on' if os.environ.get('OL_POISON') == '1' else 'off'}", flush=True)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
