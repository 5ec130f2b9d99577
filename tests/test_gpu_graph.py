"""CUDA-graph replay of repeated query shapes (option "graph", include/omniloc.h): a
replayed query returns exactly what the oracle returns for the new frames (Alg. 1 top-N,
P:95-108; Alg. 2 estimates), on the CUDA-core and tensor-core paths, for
device and host frames; options and uploads retire the graph."""
import numpy as np
import pytest
import torch

import oracle
import synthgen
import paper_2006_08861_b200 as ol
from gpu_helpers import assert_candidates_equal, assert_estimates_equal

pytestmark = pytest.mark.gpu


def _db(seed=5, paths=2, frames=1000):
    spec = synthgen.Spec(seed=seed, n_floors=1, paths=paths, frames_per_path=frames, path_y0=50.0)
    F, C = synthgen.db_host(spec)
    return spec, F, C, [frames] * paths


def _bundles(spec, seed, nb, M):
    n = nb * M + M
    video = synthgen.render_host(spec, synthgen.query_points(spec, seed, n, "path", 0, 0))["desc"]
    return np.ascontiguousarray(video[:nb * M].reshape(nb, M, -1))


@pytest.mark.parametrize("tc,nb,M", [(0, 1, 1), (0, 3, 3), (1, 64, 1)])
def test_graph_replay_matches_oracle_device_frames(tc, nb, M):
    spec, F, C, sizes = _db()
    eng = ol.Engine(0)
    eng.upload(F, C, sizes, spec.grid())
    eng.set_option("tc", tc)
    eng.set_option("graph", 1)
    qbuf = torch.empty((nb, M, 64), dtype=torch.float32, device="cuda")
    kernels = None
    for it in range(4):
        Q = _bundles(spec, 100 + it, nb, M)
        qbuf.copy_(torch.from_numpy(Q))
        eng.query(qbuf, N=5, aggregate=True)
        got, est = eng.topk(), eng.estimates()
        assert eng.stat("graph_replays") == it
        assert eng.stat("used_tc") == tc
        k = eng.stat("kernels")
        assert kernels is None or k == kernels
        kernels = k
        ref = oracle.retrieve(sizes, F, C, Q, 5)
        assert_candidates_equal(got, ref, f"iteration {it}")
        assert_estimates_equal(est, ref, ctx=f"iteration {it}")


def test_graph_replay_host_frames_and_retire():
    spec, F, C, sizes = _db(seed=9)
    eng = ol.Engine(0)
    eng.upload(F, C, sizes, spec.grid())
    eng.set_option("graph", 1)
    for it in range(3):
        Q = _bundles(spec, 200 + it, 2, 5)
        eng.query(Q, N=7, aggregate=True)
        ref = oracle.retrieve(sizes, F, C, Q, 7)
        assert_candidates_equal(eng.topk(), ref, f"host iteration {it}")
        assert_estimates_equal(eng.estimates(), ref, ctx=f"host iteration {it}")
    assert eng.stat("graph_replays") == 2
    # another shape: eager + capture, then replay
    Q = _bundles(spec, 300, 1, 5)
    eng.query(Q, N=7, aggregate=True)
    assert eng.stat("graph_replays") == 2
    # any option retires the graph: the next call runs eagerly and re-captures
    eng.set_option("graph", 1)
    eng.query(Q, N=7, aggregate=True)
    assert eng.stat("graph_replays") == 2
    eng.query(Q, N=7, aggregate=True)
    assert eng.stat("graph_replays") == 3
    ref = oracle.retrieve(sizes, F, C, Q, 7)
    assert_candidates_equal(eng.topk(), ref, "after retire")
    # a new upload retires it as well (different database, same shape)
    spec2, F2, C2, sizes2 = _db(seed=10)
    eng.upload(F2, C2, sizes2, spec2.grid())
    eng.query(Q, N=7, aggregate=True)
    assert eng.stat("graph_replays") == 3
    ref = oracle.retrieve(sizes2, F2, C2, Q, 7)
    assert_candidates_equal(eng.topk(), ref, "after upload")


def test_graph_nonfinite_frames_still_rejected():
    spec, F, C, sizes = _db(seed=11)
    eng = ol.Engine(0)
    eng.upload(F, C, sizes, spec.grid())
    eng.set_option("graph", 1)
    qbuf = torch.from_numpy(_bundles(spec, 400, 1, 1)).cuda()
    eng.query(qbuf, N=5)
    eng.query(qbuf, N=5)
    assert eng.stat("graph_replays") == 1
    qbuf[0, 0, 3] = float("nan")
    eng.query(qbuf, N=5)           # replayed: the finiteness check is part of the graph
    assert eng.stat("graph_replays") == 2
    with pytest.raises(ol.OmnilocError, match="NONFINITE"):
        eng.topk()


def test_graph_cache_alternating_shapes():
    """Micro-batches of varying size (the streaming service) each keep their own graph."""
    spec, F, C, sizes = _db(seed=12)
    eng = ol.Engine(0)
    eng.upload(F, C, sizes, spec.grid())
    eng.set_option("graph", 1)
    shapes = [1, 3, 2, 1, 3, 2, 3]
    for it, nb in enumerate(shapes):
        Q = _bundles(spec, 500 + it, nb, 5)
        eng.query(Q, N=5, aggregate=True)
        ref = oracle.retrieve(sizes, F, C, Q, 5)
        assert_candidates_equal(eng.topk(), ref, f"shape {nb} iteration {it}")
        assert_estimates_equal(eng.estimates(), ref, ctx=f"shape {nb} iteration {it}")
    # host frames go through the context buffer, which grows to 3 bundles on the second call:
    # shape 1 captured at the old buffer is re-captured once; every later call replays
    assert eng.stat("graph_replays") >= 3


def test_graph_survives_buffer_growth_elsewhere():
    """ol_aggregate on many bundles grows the estimate buffer a captured graph writes to:
    the allocation epoch retires the graph, and the next query is still exact."""
    spec, F, C, sizes = _db(seed=13)
    eng = ol.Engine(0)
    eng.upload(F, C, sizes, spec.grid())
    eng.set_option("graph", 1)
    Q = _bundles(spec, 600, 1, 3)
    eng.query(Q, N=5, aggregate=True)
    eng.query(Q, N=5, aggregate=True)
    assert eng.stat("graph_replays") == 1
    rng = np.random.default_rng(3)
    xy = rng.integers(0, 50, size=(4000, 2)).astype(np.int32)
    eng.aggregate(xy, np.arange(0, 4001, 10, dtype=np.uint32))
    Q2 = _bundles(spec, 601, 1, 3)
    eng.query(Q2, N=5, aggregate=True)
    assert eng.stat("graph_replays") == 1      # eager: the graph's buffers moved
    ref = oracle.retrieve(sizes, F, C, Q2, 5)
    assert_candidates_equal(eng.topk(), ref, "after growth")
    assert_estimates_equal(eng.estimates(), ref, ctx="after growth")
    eng.query(Q2, N=5, aggregate=True)
    assert eng.stat("graph_replays") == 2
    assert_estimates_equal(eng.estimates(), ref, ctx="replay after growth")


def test_graph_alternating_paths_and_N_on_large_db():
    """graphs of different launch layouts must not share work-item /
    chunk-range / prefix tables.  On 120k rows the CUDA-core scan (1 and 9 frames) and the
    tensor-core filter (64 frames) use different chunk sizes, and N changes the candidate
    prefix; interleaved replays of all three shapes must each stay exact (Alg. 1, P:162;
    Alg. 2)."""
    spec, F, C, sizes = _db(seed=14, paths=2, frames=60000)
    eng = ol.Engine(0)
    eng.upload(F, C, sizes, spec.grid())
    eng.set_option("graph", 1)
    shapes = [(1, 1, 5, 0), (64, 1, 15, 1), (3, 3, 7, 0)]   # (nb, M, N, expect tensor-core)
    bufs = [torch.empty((nb, M, 64), dtype=torch.float32, device="cuda") for nb, M, _, _ in shapes]
    chunks = set()
    replays = []
    for it in range(9):
        s = it % 3
        nb, M, N, tc = shapes[s]
        Q = _bundles(spec, 700 + it, nb, M)
        bufs[s].copy_(torch.from_numpy(Q))
        eng.query(bufs[s], N=N, aggregate=True)
        got, est = eng.topk(), eng.estimates()
        assert eng.stat("used_tc") == tc
        chunks.add(eng.stat("chunk"))
        replays.append(eng.stat("graph_replays"))
        ref = oracle.retrieve(sizes, F, C, Q, N)
        assert_candidates_equal(got, ref, f"shape {s} iteration {it}")
        assert_estimates_equal(est, ref, ctx=f"shape {s} iteration {it}")
    assert len(chunks) >= 2, chunks           # the shapes really use different tables
    # buffers grown by a later shape retire earlier graphs once; the last round all replays
    assert replays[6] - replays[5] == replays[7] - replays[6] == replays[8] - replays[7] == 1, replays
