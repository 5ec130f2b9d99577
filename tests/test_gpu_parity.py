"""GPU parity: the CUDA path through the C-ABI vs the CPU oracle, element by
element, bit-exact (indices, acc bits, dist bits, tiles, estimates).

Sizes: C1 and C2 in full (BASELINE configs[0], [1]); 120 random tiny DBs with
ragged subspaces, ties, duplicates, degenerate rows and flat spectra; every
coarse_k; schedule variations; logical shards; the standalone Algorithm 2;
error paths.  Full-size sampled parity for C3/C4 lives in test_gpu_fullsize.py.
"""
import numpy as np
import pytest
import torch

import oracle
import synthgen
import paper_2006_08861_b200 as ol
from gpu_helpers import assert_candidates_equal, assert_estimates_equal

pytestmark = pytest.mark.gpu

KCS = (0, 8, 16, 32)


@pytest.fixture(scope="module")
def c2():
    cfg = synthgen.CONFIGS["C2"]
    F, C = synthgen.db_host(cfg.spec)
    L = cfg.n_queries
    video = synthgen.render_host(cfg.spec, synthgen.query_points(cfg.spec, 22, L, "path", 0, 2))["desc"]
    return cfg, F, C, video


def _engine(kc=16, **opts):
    e = ol.Engine(0, coarse_k=kc)
    for k, v in opts.items():
        e.set_option(k, v)
    return e


def test_c1_full(kc=16):
    cfg = synthgen.CONFIGS["C1"]
    F, C = synthgen.db_host(cfg.spec)
    Q = synthgen.render_host(cfg.spec, synthgen.query_points(cfg.spec, 11, 1))["desc"]
    ref = oracle.retrieve(cfg.subspace_sizes, F, C, Q[:, None, :], cfg.N)
    for kc in KCS:
        e = _engine(kc)
        e.upload(F, C, cfg.subspace_sizes, cfg.spec.grid())
        e.query(Q[:, None, :], N=cfg.N, aggregate=True)
        assert_candidates_equal(e.topk(), ref, f"C1 kc={kc}")
        assert_estimates_equal(e.estimates(), ref)


@pytest.mark.parametrize("kc", KCS)
def test_c2_full_bundles_m5(c2, kc):
    cfg, F, C, video = c2
    firsts = [ol.select_window(len(video), m, cfg.M)[0] for m in range(len(video))]
    Q = synthgen.gather_windows(video, firsts, cfg.M)
    ref = oracle.retrieve(cfg.subspace_sizes, F, C, Q, cfg.N)
    e = _engine(kc)
    e.upload(torch.from_numpy(F).cuda(), torch.from_numpy(C).cuda(), cfg.subspace_sizes, cfg.spec.grid())
    e.query(torch.from_numpy(Q).cuda(), N=cfg.N, aggregate=True)
    got = e.topk()
    assert len(got) == 1000 * 5 * 5 * 15
    assert_candidates_equal(got, ref, f"C2 kc={kc}")
    if kc == 16:
        assert_estimates_equal(e.estimates(), ref)


def test_c2_m11_825_audit(c2):
    cfg, F, C, video = c2
    centres = list(range(0, len(video), 37))
    firsts = [ol.select_window(len(video), m, 11)[0] for m in centres]
    Q = synthgen.gather_windows(video, firsts, 11)
    e = _engine(16)
    e.upload(F, C, cfg.subspace_sizes, cfg.spec.grid())
    e.query(Q, N=15, aggregate=True)
    got = e.topk()
    est = e.estimates()
    assert e.candidate_count() == len(centres) * 825
    assert np.all(est["total"] == 825)
    ref = oracle.retrieve(cfg.subspace_sizes, F, C, Q, 15)
    assert_candidates_equal(got, ref, "C2 M=11")
    assert_estimates_equal(est, ref)


def _random_case(seed):
    rng = np.random.default_rng(1000 + seed)
    n_sub = int(rng.integers(1, 6))
    sizes = [int(x) for x in rng.integers(1, 301, n_sub)]
    if seed % 7 == 0:
        sizes[0] = int(rng.integers(1, 6))          # undersized subspace
    rows = sum(sizes)
    kind = seed % 3
    if kind == 0:
        F = synthgen.gflat(rows, seed=seed, dup_frac=0.05)          # flat spectra + duplicates
    elif kind == 1:
        spec = synthgen.Spec(seed=seed, n_floors=1, paths=1, frames_per_path=rows)
        F, _ = synthgen.db_host(spec)
    else:
        F = rng.random((rows, 64)).astype(np.float32)
        F[rng.integers(0, rows, max(1, rows // 20))] = 0.0          # degenerate (all-zero) rows
    C = rng.integers(0, 64, (rows, 2)).astype(np.int32)
    M = int(rng.choice([1, 3, 5, 11]))
    N = int(rng.choice([1, 5, 15, 16, 17, 64, 128]))
    B = int(rng.integers(1, 9))
    Q = F[rng.integers(0, rows, B * M)].reshape(B, M, 64).copy()
    Q[:, 0, :] += rng.standard_normal((B, 64)).astype(np.float32) * np.float32(1e-3)
    if seed % 5 == 0:
        Q[0, 0] = 0.0
    return sizes, F, C, Q, N, M


@pytest.mark.parametrize("seed", range(120))
def test_random_tiny(seed):
    sizes, F, C, Q, N, M = _random_case(seed)
    ref = oracle.retrieve(sizes, F, C, Q, N)
    kc = KCS[seed % 4]
    e = _engine(kc, chunk=[0, 64, 100, 256][seed % 4], qtile=[0, 1, 8, 24][(seed // 4) % 4])
    e.upload(F, C, sizes, (64, 64))
    agg = M * sum(min(N, s) for s in sizes) <= 8192
    e.query(Q, N=N, aggregate=agg)
    assert_candidates_equal(e.topk(), ref, f"seed {seed}")
    if agg:
        assert_estimates_equal(e.estimates(), ref, ctx=f"seed {seed}")


def test_schedule_and_hierarchy_invariance(c2):                  # S:219; R2
    cfg, F, C, video = c2
    Q = video[:300][:, None, :]
    outs = []
    for kc in KCS:
        for opts in ({}, {"tau_seed": 0}, {"chunk": 512, "qtile": 8}, {"chunk": 4000, "qtile": 64},
                     {"chunk": 1024, "qtile": 40, "tau_seed": 0}):
            e = _engine(kc, **opts)
            e.upload(F, C, cfg.subspace_sizes, cfg.spec.grid())
            e.query(Q, N=15, aggregate=True)
            outs.append((e.topk().tobytes(), e.estimates().tobytes()))
    assert all(o == outs[0] for o in outs)


@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_logical_shards_equal_single(c2, world):               # §8e sharding, one GPU
    cfg, F, C, video = c2
    Q = video[100:400][:, None, :]
    one = _engine(16)
    one.upload(F, C, cfg.subspace_sizes, cfg.spec.grid())
    one.query(Q, N=15, aggregate=True)
    want = one.topk().tobytes(), one.estimates().tobytes()
    engines, payloads = [], []
    off = np.concatenate([[0], np.cumsum(cfg.subspace_sizes)])
    for r in range(world):
        e = ol.Engine(0, coarse_k=16, rank=r, world=world, exchange="torch")
        rows = []
        for i, n in enumerate(cfg.subspace_sizes):
            b, c = ol.shard_range(n, r, world)
            rows.append(np.arange(off[i] + b, off[i] + b + c))
        rows = np.concatenate(rows)
        e.upload(F[rows], C[rows], cfg.subspace_sizes, cfg.spec.grid())
        engines.append(e)
    # per-rank queries without a process group: payloads gathered by concatenation
    for e in engines:
        e.query(Q, N=15, aggregate=True, exchange=False)
        payloads.append(e.payload())
    gathered = torch.cat(payloads)
    ref = oracle.retrieve(cfg.subspace_sizes, F, C, Q, 15)     # Alg. 1 over the whole database
    for r, e in enumerate(engines):
        e.finalize_gathered(gathered)
        got, est = e.topk(), e.estimates()
        assert_candidates_equal(got, ref, f"world {world} rank {r}")
        assert_estimates_equal(est, ref, ctx=f"world {world} rank {r}")
        assert (got.tobytes(), est.tobytes()) == want


def test_aggregate_standalone_vs_oracle():
    rng = np.random.default_rng(77)
    e = _engine(16)
    sets = []
    for s in range(200):
        n = int(rng.integers(1, 900))
        kind = s % 3
        if kind == 0:
            xy = rng.integers(0, 40, (n, 2))
        elif kind == 1:
            c = rng.integers(0, 300, (5, 2))
            xy = c[rng.integers(0, 5, n)] + rng.integers(0, 7, (n, 2))
        else:
            xy = rng.integers(0, 3000, (n, 2))
        sets.append(xy.astype(np.int32))
    off = np.concatenate([[0], np.cumsum([len(x) for x in sets])]).astype(np.uint32)
    for params in (ol.Params(), ol.Params(top_c=3, toler_per=0.5, radius_m=0.9),
                   ol.Params(top_c=64, toler_per=1.0, radius_m=1.5)):
        est = e.aggregate(np.concatenate(sets), off, params)
        for b, xy in enumerate(sets):
            r = oracle.aggregate(xy, params.top_c, params.toler_per, params.radius_m, params.tile_m)
            g = est[b]
            assert (g["x"], g["y"], bool(g["low_confidence"]), g["confidence"]) == \
                (r.x, r.y, r.low_confidence, r.confidence)
            k = int(g["n_ranked"])
            assert np.array_equal(g["ranked"]["circle"][:k], r.ranked_circle)
            assert np.array_equal(g["ranked"]["count"][:k], r.ranked_count)


def test_aggregate_small_bundles_warp_vs_block_vs_oracle():
    """Bundles of <= 32 candidates take the one-warp Algorithm 2 (aggregate_warp); option
    agg_block = 1 forces the CTA-wide version.  Both equal the oracle (ranking ties by count
    then signed (y, x), inclusive circles, the strict toler_per test and the low-confidence
    fallback) and each other byte for byte, padding of the ranked list included."""
    rng = np.random.default_rng(79)
    e = _engine(16)
    sets = []
    for s in range(400):
        n = int(rng.integers(1, 41))
        kind = s % 5
        if kind == 0:
            xy = rng.integers(0, 4, (n, 2))                              # many count ties
        elif kind == 1:
            xy = rng.integers(-6, 6, (n, 2))
        elif kind == 2:
            c = rng.integers(-50, 50, (3, 2))
            xy = c[rng.integers(0, 3, n)] + rng.integers(-2, 3, (n, 2))
        elif kind == 3:
            xy = np.repeat(rng.integers(-9, 9, (1, 2)), n, axis=0)       # one tile
        else:
            xy = rng.integers(-(1 << 30), 1 << 30, (n, 2))               # all distinct, far apart
        sets.append(xy.astype(np.int32))
    off = np.concatenate([[0], np.cumsum([len(x) for x in sets])]).astype(np.uint32)
    allxy = np.concatenate(sets)
    for params in (ol.Params(), ol.Params(top_c=3, toler_per=0.5, radius_m=0.9),
                   ol.Params(top_c=64, toler_per=1.0, radius_m=1.5), ol.Params(top_c=1, toler_per=0.05)):
        outs = []
        for block in (0, 1):
            e.set_option("agg_block", block)
            est = e.aggregate(allxy, off, params)
            outs.append(est.tobytes())
            for b, xy in enumerate(sets):
                r = oracle.aggregate(xy, params.top_c, params.toler_per, params.radius_m, params.tile_m)
                g = est[b]
                assert (g["x"], g["y"], bool(g["low_confidence"]), g["confidence"]) == \
                    (r.x, r.y, r.low_confidence, r.confidence), (b, block)
                assert g["x_m"] == r.x_m and g["y_m"] == r.y_m and int(g["total"]) == len(xy)
                k = int(g["n_ranked"])
                assert k == len(r.ranked_circle), (b, block)
                assert np.array_equal(g["ranked"]["x"][:k], r.ranked_xy[:, 0]), (b, block)
                assert np.array_equal(g["ranked"]["y"][:k], r.ranked_xy[:, 1]), (b, block)
                assert np.array_equal(g["ranked"]["circle"][:k], r.ranked_circle), (b, block)
                assert np.array_equal(g["ranked"]["count"][:k], r.ranked_count), (b, block)
                assert not g["ranked"][k:].tobytes().strip(b"\0"), (b, block)
        assert outs[0] == outs[1]
    e.set_option("agg_block", 0)


def test_micro_kernel_split_shares_vs_oracle():
    """NK10 splits each (frame, subspace) job over several CTAs (shares of >= 256 rows, the
    last CTA merges the shares' lists): subspaces of 1..8,192 rows, N up to 128 (a 1,024-key
    merge), bundles of several jobs, against the oracle; the block-wide Alg. 2 agrees."""
    rng = np.random.default_rng(950)
    for case in range(6):
        sizes = [[8192], [8000, 3], [257, 255, 1], [2000], [4097, 4096], [600, 700, 800]][case]
        F = np.abs(rng.standard_normal((sum(sizes), 64))).astype(np.float32)
        F /= np.linalg.norm(F, axis=1, keepdims=True)
        F[rng.integers(0, len(F), 30)] = F[rng.integers(0, len(F), 30)]   # exact duplicates: ties
        C = rng.integers(0, 60, (sum(sizes), 2)).astype(np.int32)
        M = [1, 1, 3, 1, 1, 5][case]
        nb = max(1, (1 << 16) // (len(F) * M))
        nb = min(nb, 3)
        Q = (F[rng.integers(0, len(F), nb * M)] + 1e-3 * rng.standard_normal((nb * M, 64))).astype(np.float32)
        Q = np.ascontiguousarray(Q.reshape(nb, M, 64))
        for N in ([128, 15] if case < 2 else [5, 40]):
            ref = oracle.retrieve(sizes, F, C, Q, N)
            e = _engine(16)
            e.upload(F, C, sizes, (64, 64))
            outs = []
            for block in (0, 1):
                e.set_option("agg_block", block)
                e.query(Q, N=N, aggregate=True)
                assert e.stat("used_micro") == 1 and e.stat("kernels") == 1
                got, est = e.topk(), e.estimates()
                assert_candidates_equal(got, ref, f"split case {case} N {N}")
                assert_estimates_equal(est, ref, ctx=f"split case {case} N {N}")
                outs.append((got.tobytes(), est.tobytes()))
            assert outs[0] == outs[1]
            e.close()


@pytest.mark.parametrize("tc", [0, 1])
def test_merge_gather_and_fallback_vs_oracle(tc):
    """The per-rank merge gathers only the keys <= min over work-item lists of list[N-1] (the
    lists are ascending); option merge_scan = 1 takes its fallback, N rounds of a CTA-wide
    minimum over every key.  Both equal the oracle with many lists per subspace (small
    chunks), ragged subspaces, N above and below 32, and ties from duplicated rows."""
    rng = np.random.default_rng(960 + tc)
    sizes = [9000, 6001, 40]
    F = np.abs(rng.standard_normal((sum(sizes), 64))).astype(np.float32)
    F /= np.linalg.norm(F, axis=1, keepdims=True)
    F[rng.integers(0, len(F), 50)] = F[rng.integers(0, len(F), 50)]
    C = rng.integers(0, 60, (sum(sizes), 2)).astype(np.int32)
    Q = (F[rng.integers(0, len(F), 60)] + 1e-3 * rng.standard_normal((60, 64))).astype(np.float32)
    Q = np.ascontiguousarray(Q.reshape(20, 3, 64))
    for N in (15, 40):
        ref = oracle.retrieve(sizes, F, C, Q, N)
        outs = []
        for scan in (0, 1):
            e = _engine(16, tc=tc, chunk=512, merge_scan=scan)
            e.upload(F, C, sizes, (64, 64))
            e.query(Q, N=N, aggregate=True)
            assert e.stat("used_tc") == tc and e.stat("items") >= 30
            assert_candidates_equal(e.topk(), ref, f"merge tc {tc} N {N} scan {scan}")
            assert_estimates_equal(e.estimates(), ref, ctx=f"merge tc {tc} N {N} scan {scan}")
            outs.append(e.topk().tobytes())
            e.close()
        assert outs[0] == outs[1]


def test_seed_select_gather_warp_vs_other_selects_vs_oracle():
    """The two-kernel seed's warp-per-job select (samples <= 4,096: N-th smallest of a strided
    subset as the bound, one gathering pass, sorting networks) finds the same thresholds as
    the CTA / radix selects (option seed_select = 1) -- the exact N-th smallest of every
    job's samples -- including a subspace of identical rows (every sample ties, the gather
    buffer overflows), N above and below 16; the queries then equal the oracle."""
    rng = np.random.default_rng(990)
    sizes = [33000, 40000, 33000, 36001, 32768]
    F = np.abs(rng.standard_normal((sum(sizes), 64))).astype(np.float32)
    F /= np.linalg.norm(F, axis=1, keepdims=True)
    F[73000:106000] = F[73000]                                   # subspace 2: one row repeated
    C = rng.integers(0, 60, (sum(sizes), 2)).astype(np.int32)
    Q = (F[rng.integers(0, len(F), 40)] + 1e-3 * rng.standard_normal((40, 64))).astype(np.float32)
    Q = np.ascontiguousarray(Q.reshape(40, 1, 64))
    for N, S in ((15, 4096), (15, 2500), (31, 300), (5, 64)):
        taus = []
        for sel in (0, 1):
            e = _engine(16, tc_seed=0, seed_samples=S, seed_select=sel, tc_debug=512)
            e.upload(F, C, sizes, (64, 64))
            e.query(Q, N=N)
            taus.append(e.thresholds().cpu().numpy().copy())
            e.close()
        assert (taus[0] == taus[1]).all(), f"N {N} S {S}: thresholds differ"
        assert (taus[0] < 0x7F800000).all()                     # every job seeded
        e = _engine(16, tc_seed=0, seed_samples=S)
        e.upload(F, C, sizes, (64, 64))
        e.query(Q, N=N)
        assert_candidates_equal(e.topk(), oracle.retrieve(sizes, F, C, Q, N), f"seed select N {N} S {S}")
        e.close()


@pytest.mark.parametrize("kc", [0, 8, 16, 32, 64])
def test_small_batch_cuda_core_kernels_vs_oracle(kc):
    """The CUDA-core scans for few frames -- scan3 (TMA-fed; automatic for 1-2 frames per tile),
    scan2 (row-pair streaming; automatic up to 16) and the general scan_kernel (option
    scan2 = 0) -- equal the oracle for every coarse width, 1 to 16 frames, ragged subspaces."""
    rng = np.random.default_rng(970 + kc)
    sizes = [12001, 9000, 37]
    F = np.abs(rng.standard_normal((sum(sizes), 64))).astype(np.float32)
    F /= np.linalg.norm(F, axis=1, keepdims=True)
    F[rng.integers(0, len(F), 40)] = F[rng.integers(0, len(F), 40)]
    C = rng.integers(0, 60, (sum(sizes), 2)).astype(np.int32)
    for chunk in (0, 100):   # (100: work items off the 32-row tiles -- scan3 then stands aside)
        e = _engine(kc, tc=0, micro=0, chunk=chunk)
        e.upload(F, C, sizes, (64, 64))
        for nq in (1, 2, 5, 16):
            Q = (F[rng.integers(0, len(F), nq)] + 1e-3 * rng.standard_normal((nq, 64))).astype(np.float32)
            Q = np.ascontiguousarray(Q.reshape(nq, 1, 64))
            ref = oracle.retrieve(sizes, F, C, Q, 15)
            for v in (1, 2, 0):
                e.set_option("scan2", v)
                e.query(Q, N=15, aggregate=True)
                assert e.stat("used_tc") == 0
                ctx = f"kc {kc} chunk {chunk} nq {nq} scan2 {v}"
                assert_candidates_equal(e.topk(), ref, ctx)
                assert_estimates_equal(e.estimates(), ref, ctx=ctx)


def test_aggregate_negative_tiles_and_grid_range():
    """Standalone Alg. 2 ranks tiles by count, then signed (y, x) ascending (R7) for
    any tile, negative ones included (the unbiased sort key put them last);
    with a database uploaded, tiles outside its grid are rejected."""
    rng = np.random.default_rng(78)
    e = _engine(16)
    sets = []
    for s in range(120):
        n = int(rng.integers(1, 400))
        kind = s % 4
        if kind == 0:      # ties across the sign boundary: equal counts at (-1, y) and (1, y)
            base = np.array([[-1, -1], [1, -1], [-1, 1], [1, 1], [0, 0]])
            xy = base[rng.integers(0, 5, n)]
        elif kind == 1:
            xy = rng.integers(-40, 40, (n, 2))
        elif kind == 2:
            xy = rng.integers(-(1 << 30), (1 << 30), (n, 2))
        else:
            c = rng.integers(-300, 300, (4, 2))
            xy = c[rng.integers(0, 4, n)] + rng.integers(-5, 6, (n, 2))
        sets.append(xy.astype(np.int32))
    off = np.concatenate([[0], np.cumsum([len(x) for x in sets])]).astype(np.uint32)
    allxy = np.concatenate(sets)
    for params in (ol.Params(), ol.Params(top_c=64, toler_per=0.9, radius_m=0.6)):
        for dev in (False, True):
            if dev:
                est = e.aggregate(torch.from_numpy(allxy).cuda(), torch.from_numpy(off.astype(np.int32)).cuda(),
                                  params)
            else:
                est = e.aggregate(allxy, off, params)
            for b, xy in enumerate(sets):
                r = oracle.aggregate(xy, params.top_c, params.toler_per, params.radius_m, params.tile_m)
                g = est[b]
                assert (g["x"], g["y"], bool(g["low_confidence"]), g["confidence"]) == \
                    (r.x, r.y, r.low_confidence, r.confidence), (b, dev)
                assert g["x_m"] == r.x_m and g["y_m"] == r.y_m
                k = int(g["n_ranked"])
                assert np.array_equal(g["ranked"]["x"][:k], r.ranked_xy[:, 0]), (b, dev)
                assert np.array_equal(g["ranked"]["y"][:k], r.ranked_xy[:, 1]), (b, dev)
                assert np.array_equal(g["ranked"]["count"][:k], r.ranked_count)
                assert np.array_equal(g["ranked"]["circle"][:k], r.ranked_circle)
    # outside the int32 safety range (no database): rejected, host and device
    big = np.array([[1 << 30, 0]], np.int32)
    with pytest.raises(ol.OmnilocError, match="OUT_OF_RANGE"):
        e.aggregate(big, np.array([0, 1], np.uint32))
    with pytest.raises(ol.OmnilocError, match="OUT_OF_RANGE"):
        e.aggregate(torch.from_numpy(big).cuda(), torch.tensor([0, 1], dtype=torch.int32, device="cuda"))
    # with a database: its grid bounds the tiles
    cfg = synthgen.CONFIGS["C1"]
    F, C = synthgen.db_host(cfg.spec)
    e.upload(F, C, cfg.subspace_sizes, cfg.spec.grid())
    gw, gh = cfg.spec.grid()
    for bad in ([-1, 0], [0, -1], [gw, 0], [0, gh]):
        xy = np.array([[1, 1], bad], np.int32)
        with pytest.raises(ol.OmnilocError, match="OUT_OF_RANGE"):
            e.aggregate(xy, np.array([0, 2], np.uint32))
        with pytest.raises(ol.OmnilocError, match="OUT_OF_RANGE"):
            e.aggregate(torch.from_numpy(xy).cuda(), torch.tensor([0, 2], dtype=torch.int32, device="cuda"))
    ok = np.array([[0, 0], [gw - 1, gh - 1]], np.int32)
    est = e.aggregate(ok, np.array([0, 2], np.uint32))
    r = oracle.aggregate(ok)
    assert (est[0]["x"], est[0]["y"]) == (r.x, r.y)


def test_error_paths():
    cfg = synthgen.CONFIGS["C1"]
    F, C = synthgen.db_host(cfg.spec)
    e = _engine(16)
    with pytest.raises(ol.OmnilocError, match="NOT_READY"):
        e.query(F[:1][:, None, :], N=5)
    bad = F.copy(); bad[3, 5] = np.nan
    with pytest.raises(ol.OmnilocError, match="NONFINITE"):
        e.upload(bad, C, [2000], cfg.spec.grid())
    with pytest.raises(ol.OmnilocError, match="OUT_OF_RANGE"):
        e.upload(F, C, [2000], (10, 10))
    e.upload(F, C, [2000], cfg.spec.grid())
    q = F[:1][:, None, :].copy(); q[0, 0, 0] = np.inf
    with pytest.raises(ol.OmnilocError, match="NONFINITE"):
        e.query(q, N=5)
    qd = torch.from_numpy(q).cuda()
    e.query(qd, N=5)
    with pytest.raises(ol.OmnilocError, match="NONFINITE"):
        e.topk()
    for kw in ({"N": 0}, {"N": 129}):
        with pytest.raises(ol.OmnilocError, match="INVALID"):
            e.query(F[:1][:, None, :], **kw)
    with pytest.raises(ol.OmnilocError, match="INVALID"):
        e.query(F[:2].reshape(1, 2, 64), N=5)          # M even
    with pytest.raises(ol.OmnilocError, match="INVALID"):
        e.query(F[:1][:, None, :], N=5, params=ol.Params(5, 10, 0.0, 3.0, 0.3))
    with pytest.raises(ol.OmnilocError, match="EMPTY"):
        e.aggregate(np.zeros((3, 2), np.int32), np.array([0, 3, 3], np.uint32))
    e.query(F[:1][:, None, :], N=5, aggregate=False)
    with pytest.raises(ol.OmnilocError, match="EMPTY"):
        e.estimates()


@pytest.mark.parametrize("world", [2, 3, 8])
def test_p2p_exchange_emulated_equals_single(c2, world):        # §8e, the peer-memory exchange
    """The fused exchange + merge kernel (ol_p2p_*), `world` ranks emulated on one GPU
    by one cooperative launch: every rank's candidates and estimates equal the W = 1
    answer, over consecutive queries of different sizes (mailbox double-buffering,
    monotonic arrival counters) and a mailbox re-open."""
    cfg, F, C, video = c2
    off = np.concatenate([[0], np.cumsum(cfg.subspace_sizes)])
    engines = []
    for r in range(world):
        e = ol.Engine(0, coarse_k=16, rank=r, world=world, exchange="torch")
        rows = np.concatenate([np.arange(off[i] + b, off[i] + b + c) for i, n in enumerate(cfg.subspace_sizes)
                               for b, c in [ol.shard_range(n, r, world)]])
        e.upload(F[rows], C[rows], cfg.subspace_sizes, cfg.spec.grid())
        engines.append(e)
    one = _engine(16)
    one.upload(F, C, cfg.subspace_sizes, cfg.spec.grid())
    cap = 300 * len(cfg.subspace_sizes) * 15 * 16
    for r, e in enumerate(engines):
        assert len(e.p2p_open(world, r, cap)) == 64
    for it, (a, b) in enumerate([(100, 400), (0, 37), (500, 800), (7, 8), (200, 500)]):
        Q = video[a:b][:, None, :]
        one.query(Q, N=15, aggregate=True)
        want = one.topk().tobytes(), one.estimates().tobytes()
        for e in engines:
            e.query(Q, N=15, aggregate=True, exchange=False)
        ol.p2p_emulate(engines)
        ref = oracle.retrieve(cfg.subspace_sizes, F, C, Q, 15)
        for r, e in enumerate(engines):
            got, est = e.topk(), e.estimates()
            assert_candidates_equal(got, ref, f"query {it} rank {r}")
            assert_estimates_equal(est, ref, ctx=f"query {it} rank {r}")
            assert (got.tobytes(), est.tobytes()) == want, f"query {it} rank {r}"
        if it == 2:   # a re-open (new mailboxes, epochs restart)
            for r, e in enumerate(engines):
                e.p2p_open(world, r, cap * 2)
    # a payload larger than the mailbox is refused
    Q = video[:400][:, None, :]
    for e in engines:
        e.query(Q, N=15, aggregate=True, exchange=False)
    with pytest.raises(ol.OmnilocError):
        engines[0].p2p_open(world, 0, 16)
        ol.p2p_emulate(engines)


@pytest.mark.parametrize("world", [2, 4])
def test_tau_share_emulated_shards_match_oracle(c2, world):        # §8e, in-scan threshold sharing
    """Ranks that MIN their published thresholds into each other's arrays during the scan (NCCL
    mode over peer memory; here `world` contexts on one GPU linked by ol_tau_share_emulate,
    their queries running concurrently on separate streams) still return exactly the oracle's
    top-N and estimates: any rank's threshold bounds the global N-th best (Alg. 1)."""
    cfg, F, C, video = c2
    off = np.concatenate([[0], np.cumsum(cfg.subspace_sizes)])
    engines, streams = [], []
    for r in range(world):
        st = torch.cuda.Stream()
        e = ol.Engine(0, coarse_k=16, rank=r, world=world, exchange="torch", stream=st)
        e.set_option("tc", 1)
        rows = np.concatenate([np.arange(off[i] + b, off[i] + b + c) for i, n in enumerate(cfg.subspace_sizes)
                               for b, c in [ol.shard_range(n, r, world)]])
        e.upload(F[rows], C[rows], cfg.subspace_sizes, cfg.spec.grid())
        engines.append(e); streams.append(st)
    Qs = [np.ascontiguousarray(video[a:a + 300][:, None, :]) for a in (0, 300, 600)]
    Qd = [torch.from_numpy(q).cuda() for q in Qs]
    torch.cuda.synchronize()
    for e in engines:                      # every context allocates this shape's arrays first
        e.query(Qd[0], N=15, aggregate=True, exchange=False)
    torch.cuda.synchronize()
    ol.tau_share_emulate(engines)
    for k, q in enumerate(Qd):
        for e in engines:                  # all ranks' scans in flight at once
            e.query(q, N=15, aggregate=True, exchange=False)
        assert all(e.stat("tau_peers") == world - 1 for e in engines)
        pays = [e.payload() for e in engines]
        torch.cuda.synchronize()
        g = torch.cat(pays)
        torch.cuda.synchronize()
        ref = oracle.retrieve(cfg.subspace_sizes, F, C, Qs[k], 15)
        for r, e in enumerate(engines):
            e.finalize_gathered(g)
            assert_candidates_equal(e.topk(), ref, f"tau share world {world} query {k} rank {r}")
            assert_estimates_equal(e.estimates(), ref, ctx=f"tau share world {world} query {k} rank {r}")
    e = engines.pop()
    e.close()                              # unlinks itself from the others
    assert engines[0].stat("tau_peers") == world - 2


@pytest.mark.parametrize("seed", range(6))
def test_micro_kernel_small_queries_vs_oracle(seed):            # NK10, the latency configurations
    """Small world-1 queries run as ONE kernel (scan, top-N, candidate rows, Alg. 2 by each
    bundle's last job): candidates and estimates equal the oracle's, with several subspaces
    (one smaller than N), bundles of M = 1/3/5, ties from duplicated rows, and graph
    replay; the same queries with the kernel disabled give the same bytes."""
    rng = np.random.default_rng(900 + seed)
    sizes = [int(rng.integers(2, 3000)) for _ in range(int(rng.integers(1, 4)))]
    sizes[0] = min(sizes[0], 9)                                   # an undersized subspace
    F = np.abs(rng.standard_normal((sum(sizes), 64))).astype(np.float32)
    F /= np.linalg.norm(F, axis=1, keepdims=True)
    F[rng.integers(0, len(F), 20)] = F[rng.integers(0, len(F), 20)]   # exact duplicates: ties
    C = rng.integers(0, 60, (sum(sizes), 2)).astype(np.int32)
    M = int(rng.choice([1, 3, 5]))
    nb = int(rng.integers(1, 6))
    nb = max(1, min(nb, (1 << 16) // (len(F) * M)))   # within the single-kernel size
    M = M if nb * M * len(F) <= (1 << 16) else 1
    Q = (F[rng.integers(0, len(F), nb * M)] + 1e-3 * rng.standard_normal((nb * M, 64))).astype(np.float32)
    Q = np.ascontiguousarray(Q.reshape(nb, M, 64))
    N = int(rng.choice([1, 5, 15, 40]))
    ref = oracle.retrieve(sizes, F, C, Q, N)
    e = _engine(16)
    e.upload(F, C, sizes, (64, 64))
    e.query(Q, N=N, aggregate=True)
    assert e.stat("used_micro") == 1 and e.stat("kernels") == 1
    got, est = e.topk(), e.estimates()
    assert_candidates_equal(got, ref, f"micro seed {seed}")
    assert_estimates_equal(est, ref, ctx=f"micro seed {seed}")
    e.set_option("graph", 1)
    qd = torch.from_numpy(Q).cuda()
    for _ in range(3):
        e.query(qd, N=N, aggregate=True)
    assert e.stat("graph_replays") == 2 and e.stat("used_micro") == 1
    assert e.topk().tobytes() == got.tobytes() and e.estimates().tobytes() == est.tobytes()
    e.set_option("graph", 0)
    e.set_option("micro", 0)
    e.query(Q, N=N, aggregate=True)
    assert e.stat("used_micro") == 0
    assert e.topk().tobytes() == got.tobytes() and e.estimates().tobytes() == est.tobytes()


def test_get_results_one_fetch():
    """ol_get_results copies the candidates and the estimates with one synchronisation: the
    same bytes as ol_get_topk + ol_get_estimates; EMPTY when estimates are asked of a query
    that did not aggregate; INVALID_ARGUMENT for short buffers."""
    import torch
    cfg = synthgen.CONFIGS["C1"]
    F, C = synthgen.db_host(cfg.spec)
    Q = synthgen.render_host(cfg.spec, synthgen.query_points(cfg.spec, 11, 3))["desc"][:, None, :]
    e = _engine(16)
    e.upload(F, C, cfg.subspace_sizes, cfg.spec.grid())
    e.query(Q, N=cfg.N, aggregate=True)
    got, est = e.topk(), e.estimates()
    res = torch.empty(len(got) * ol.CANDIDATE_DTYPE.itemsize, dtype=torch.uint8)
    es = torch.empty(len(est) * ol.ESTIMATE_DTYPE.itemsize, dtype=torch.uint8)
    nb, ne = e.results_into(res, es)
    assert nb == res.numel() and ne == es.numel()
    assert res.numpy().tobytes() == got.tobytes() and es.numpy().tobytes() == est.tobytes()
    assert e.results_into(res)[0] == res.numel()                      # candidates only
    with pytest.raises(ol.OmnilocError, match="INVALID_ARGUMENT"):
        e.results_into(res[: res.numel() - 1], es)
    e.query(Q, N=cfg.N, aggregate=False)
    with pytest.raises(ol.OmnilocError, match="EMPTY"):
        e.results_into(res, es)
