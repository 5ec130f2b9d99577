"""GPU parity of the tensor-core certified filter (tcscan, NEXT-2): forced on and
off, bit-exact against the oracle on paper-shaped data, flat spectra, negative
and degenerate vectors, many subspaces, large N (smaller query blocks), values
outside the fp16 range (the library must fall back to the CUDA-core scan), and
without threshold seeding (every pair survives until the lists fill)."""
import numpy as np
import pytest

import oracle
import synthgen
import paper_2006_08861_b200 as ol
from gpu_helpers import assert_candidates_equal, assert_estimates_equal

pytestmark = pytest.mark.gpu


def _run(F, C, sizes, Q, N, tc, grid=(4096, 4096), agg=True, **opts):
    e = ol.Engine(0, coarse_k=16)
    e.set_option("tc", tc)
    for k, v in opts.items():
        e.set_option(k, v)
    e.upload(F, C, sizes, grid)
    e.query(Q, N=N, aggregate=agg)
    return e


@pytest.mark.parametrize("N", [1, 15, 64, 128])
def test_tc_paper_shaped(N):
    spec = synthgen.Spec(seed=31, n_floors=2, paths=5, frames_per_path=1200)
    F, C = synthgen.db_host(spec)
    Q = synthgen.render_host(spec, synthgen.query_points(spec, 9, 300))["desc"][:, None, :]
    ref = oracle.retrieve([F.shape[0]], F, C, Q, N)
    for tc in (1, 0):
        e = _run(F, C, [F.shape[0]], Q, N, tc, spec.grid())
        # lists of N = 128 may leave too little shared memory for the tensor-core
        # pipeline (then: CUDA-core scan); results are identical either way
        assert e.stat("used_tc") == tc if N < 128 else e.stat("used_tc") in (0, tc)
        assert_candidates_equal(e.topk(), ref, f"N={N} tc={tc}")
        if tc and N <= 15:
            assert e.stat("survivors") < 0.02 * e.stat("pairs")


@pytest.mark.parametrize("seed", range(12))
def test_tc_adversarial(seed):
    rng = np.random.default_rng(500 + seed)
    sizes = [int(x) for x in rng.integers(50, 3000, int(rng.integers(1, 4)))]
    rows = sum(sizes)
    kind = seed % 4
    if kind == 0:
        F = synthgen.gflat(rows, seed=seed, dup_frac=0.05)
    elif kind == 1:
        F = (rng.standard_normal((rows, 64)) * 3).astype(np.float32)      # signed, non-unit
    elif kind == 2:
        F = rng.random((rows, 64)).astype(np.float32)
        F[rng.integers(0, rows, rows // 10)] = 0.0                        # degenerate rows
    else:
        F = (rng.random((rows, 64)) * 1e-3).astype(np.float32)             # fp16 subnormal range
    C = rng.integers(0, 500, (rows, 2)).astype(np.int32)
    M = int(rng.choice([1, 3, 5]))
    B = int(rng.integers(8, 80))
    Q = F[rng.integers(0, rows, B * M)].reshape(B, M, 64).copy()
    Q += (rng.standard_normal(Q.shape) * 1e-4).astype(np.float32)
    Q[0, 0] = 0.0
    N = int(rng.choice([5, 15, 33]))
    ref = oracle.retrieve(sizes, F, C, Q, N)
    opts = {"tau_seed": 0} if seed % 3 == 0 else {}
    opts["inline_rescore"] = [-1, 0][seed % 2]   # (small databases default to inline re-scoring)
    e = _run(F, C, sizes, Q, N, 1, **opts)
    assert e.stat("used_tc") == 1
    assert_candidates_equal(e.topk(), ref, f"seed {seed}")
    assert_estimates_equal(e.estimates(), ref, ctx=f"seed {seed}")


def test_tc_out_of_fp16_range_falls_back():
    rng = np.random.default_rng(9)
    F = rng.random((3000, 64)).astype(np.float32)
    F[17, 3] = 1e6
    C = rng.integers(0, 100, (3000, 2)).astype(np.int32)
    Q = F[:40][:, None, :].copy()
    ref = oracle.retrieve([3000], F, C, Q, 15)
    e = _run(F, C, [3000], Q, 15, 1)
    assert e.stat("tc_ok") == 0 and e.stat("used_tc") == 0
    assert_candidates_equal(e.topk(), ref, "fallback")
    # a query out of range: still the TC kernel, every pair re-scored exactly
    Q2 = Q.copy()
    Q2[3, 0, 5] = 7e4
    F2 = F.copy(); F2[17, 3] = 0.5
    ref2 = oracle.retrieve([3000], F2, C, Q2, 15)
    e2 = _run(F2, C, [3000], Q2, 15, 1)
    assert e2.stat("used_tc") == 1
    assert_candidates_equal(e2.topk(), ref2, "query out of range")


def test_tc_schedule_invariance():
    spec = synthgen.Spec(seed=33, n_floors=1, paths=5, frames_per_path=2000)
    F, C = synthgen.db_host(spec)
    Q = synthgen.render_host(spec, synthgen.query_points(spec, 5, 600))["desc"][:, None, :]
    outs = set()
    for opts in ({}, {"chunk": 4096}, {"chunk": 128}, {"tau_seed": 0, "chunk": 2048}, {"tc": 0}):
        e = ol.Engine(0)
        e.set_option("tc", 1)
        for k, v in opts.items():
            e.set_option(k, v)
        e.upload(F, C, [F.shape[0]], spec.grid())
        e.query(Q, N=15)
        outs.add(e.topk().tobytes() + e.estimates().tobytes())
    assert len(outs) == 1


@pytest.mark.parametrize("kind", ["paper", "signed"])
def test_tc_bound_prepass_seed(kind):
    """The tensor-core bound pre-pass (tau seed from certified upper bounds of every S-th
    row's tensor-core score) only changes thresholds: results stay bit-identical to the
    oracle, with the pre-pass on or off, over 2 subspaces large enough to use it."""
    # (the pre-pass runs when every subspace has >= 256 N rows in its 1/64 sample)
    if kind == "paper":
        spec = synthgen.Spec(seed=33, n_floors=26, paths=5, frames_per_path=4000)   # 520k rows
        F, C = synthgen.db_host(spec)
        Q = synthgen.render_host(spec, synthgen.query_points(spec, 19, 160))["desc"][:, None, :]
    else:
        rng = np.random.default_rng(33)
        F = (rng.standard_normal((520_000, 64)) * 2).astype(np.float32)     # signed, non-unit
        C = rng.integers(0, 500, (520_000, 2)).astype(np.int32)
        Q = (F[rng.integers(0, 520_000, 160)] + rng.standard_normal((160, 64)).astype(np.float32) * 0.05)[:, None, :]
    sizes = [260_000, 260_000]
    N = 15
    grid = spec.grid() if kind == "paper" else (4096, 4096)
    outs = []
    for ts in (1, 0):
        e = _run(F, C, sizes, Q, N, 1, grid=grid, agg=False, tc_seed=ts)
        assert e.stat("used_tc") == 1
        outs.append(e.topk())
    assert np.array_equal(outs[0], outs[1])
    sub = np.arange(0, 160, 8)
    ref = oracle.retrieve(sizes, F, C, Q[sub], N)
    got = outs[0].reshape(160, -1)[sub].reshape(-1)
    assert np.array_equal(got["frame"], ref.frame) and np.array_equal(got["subspace"], ref.subspace)
    assert np.array_equal(got["dist2"].view(np.uint32), ref.acc.view(np.uint32))


@pytest.mark.parametrize("nq", [256, 600, 647])
def test_tc_cta_pairs(nq):
    """CTA pairs (tcgen05 cta_group::2, M = 256 over two query blocks, each CTA loading half
    of every row tile): identical results to single CTAs and to the oracle, including an odd
    number of query blocks (600 frames = 5 blocks: a padding CTA), a ragged last query block
    (647) and a ragged last row tile."""
    spec = synthgen.Spec(seed=34, n_floors=2, paths=5, frames_per_path=1207)
    F, C = synthgen.db_host(spec)
    Q = synthgen.render_host(spec, synthgen.query_points(spec, 21, nq))["desc"][:, None, :]
    sizes = [7000, F.shape[0] - 7000]
    outs = []
    for pair in (2, 0):
        e = _run(F, C, sizes, Q, 15, 1, agg=False, pair=pair)
        assert e.stat("used_tc") == 1 and e.stat("used_pair") == (pair == 2)
        outs.append(e.topk())
    assert np.array_equal(outs[0], outs[1])
    ref = oracle.retrieve(sizes, F, C, Q, 15)
    assert_candidates_equal(outs[0], ref, f"pair nq={nq}")


@pytest.mark.parametrize("kf", [16, 32, 48])
def test_tc_prefix_filter(kf):
    """Option tc_k: the certified filter on the first kf dimensions only (the prefix
    distance is a lower bound of the full one, so pruning stays exact): bit-identical
    to the oracle and to the full-K filter, with pairs and single CTAs."""
    spec = synthgen.Spec(seed=36, n_floors=2, paths=5, frames_per_path=1207)
    F, C = synthgen.db_host(spec)
    Q = synthgen.render_host(spec, synthgen.query_points(spec, 25, 600))["desc"][:, None, :]
    sizes = [7000, F.shape[0] - 7000]
    ref = oracle.retrieve(sizes, F, C, Q, 15)
    for pair in (2, 0):
        e = _run(F, C, sizes, Q, 15, 1, agg=False, pair=pair, tc_k=kf)
        assert e.stat("used_tc") == 1
        assert_candidates_equal(e.topk(), ref, f"tc_k={kf} pair={pair}")
    rng = np.random.default_rng(kf)
    G = (rng.standard_normal((5000, 64)) * 2).astype(np.float32)      # signed, non-unit
    CG = rng.integers(0, 500, (5000, 2)).astype(np.int32)
    QG = (G[rng.integers(0, 5000, 200)] + rng.standard_normal((200, 64)).astype(np.float32) * 0.05)[:, None, :]
    e = _run(G, CG, [5000], QG, 15, 1, agg=False, tc_k=kf)
    assert_candidates_equal(e.topk(), oracle.retrieve([5000], G, CG, QG, 15), f"tc_k={kf} signed")


@pytest.mark.parametrize("N,nq", [(64, 300), (128, 130), (1, 7)])
def test_tc_narrow_plane_large_and_small_N(N, nq):
    """The 64-B fp16 plane (tc_k = 32): deeper pipelines fit next to large top-N lists (N up to
    128), and few frames (7: epilogue warps without frames skip their TMEM reads)."""
    spec = synthgen.Spec(seed=37, n_floors=2, paths=5, frames_per_path=1000)
    F, C = synthgen.db_host(spec)
    Q = synthgen.render_host(spec, synthgen.query_points(spec, 27, nq))["desc"][:, None, :]
    sizes = [6000, F.shape[0] - 6000]
    ref = oracle.retrieve(sizes, F, C, Q, N)
    for pair in (2, 0):
        e = _run(F, C, sizes, Q, N, 1, agg=False, pair=pair, tc_k=32)
        assert e.stat("used_tc") == 1 and e.stat("tc_k") == 32
        assert_candidates_equal(e.topk(), ref, f"N={N} nq={nq} pair={pair}")


@pytest.mark.parametrize("N", [5, 15, 40, 128])
def test_tc_inline_rescore(N):
    """Short work items (C2-like: a small database, many frames) re-score survivors in the
    epilogue warps themselves (per-frame list locks; option inline_rescore, automatic for work
    subspaces averaging <= 65,536 rows); forced on and off, on paper-shaped and adversarial (flat-spectrum,
    duplicated) data, the results equal the oracle."""
    spec = synthgen.Spec(seed=77, n_floors=1, paths=5, frames_per_path=900)
    F, C = synthgen.db_host(spec)
    sizes = [900] * 5
    V = synthgen.render_host(spec, synthgen.query_points(spec, 13, 700))["desc"]
    Q = np.ascontiguousarray(V[:695].reshape(139, 5, 64))
    G = synthgen.gflat(3000, seed=5, dup_frac=0.1)
    Cg = np.random.default_rng(6).integers(0, 500, (3000, 2)).astype(np.int32)
    Qg = np.ascontiguousarray((G[np.random.default_rng(7).integers(0, 3000, 300)] + 1e-3).astype(np.float32).reshape(300, 1, 64))
    for (FF, CC, ss, QQ, grid) in ((F, C, sizes, Q, spec.grid()), (G, Cg, [1000, 2000], Qg, (4096, 4096))):
        ref = oracle.retrieve(ss, FF, CC, QQ, N)
        for v in (1, 0, -1):
            e = _run(FF, CC, ss, QQ, N, 1, grid, inline_rescore=v)
            assert e.stat("used_tc") == 1 or N == 128
            assert_candidates_equal(e.topk(), ref, f"N={N} inline={v}")
            assert_estimates_equal(e.estimates(), ref, ctx=f"N={N} inline={v}")
            e.close()
