"""Pins for the oracle's top-N retrieval and window helper (CPU only).

External pins: Python's own sort on (acc, index), the cardinality law
(S:220), the 825-candidate count of the paper, SPEC's window
examples, self-retrieval at distance +0, undersized
subspaces and adjacency of duplicates.
"""
import json
import os

import numpy as np
import pytest

import oracle
import synthgen

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _python_topn(acc, N):
    order = sorted(range(len(acc)), key=lambda t: (float(acc[t]), t))[:N]
    return np.array(order, np.uint32)


@pytest.mark.parametrize("seed", range(8))
def test_topn_sortall_and_select_equal_python_sort(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 400))
    # heavy ties: values drawn from a small set
    acc = rng.choice(np.float32([0, 0.5, 0.25, 1e-3, 2.0, 0.125]), n).astype(np.float32)
    if seed % 2:
        acc = rng.random(n).astype(np.float32)
    for N in (1, 5, 15, 16, 17, 64, 128, 500):
        exp = _python_topn(acc, N)
        for method in ("sortall", "select"):
            idx, a = oracle.topn(acc, N, method)
            assert np.array_equal(idx, exp), (method, N)
            assert np.array_equal(a, acc[exp])


def _tiny_db(rng, n_sub, sizes, K=64, dup=True):
    F = np.abs(rng.standard_normal((sum(sizes), K))).astype(np.float32)
    F /= np.linalg.norm(F, axis=1, keepdims=True)
    if dup and F.shape[0] > 4:
        F[3] = F[1]
        F[-1] = F[1]
    C = rng.integers(0, 50, (sum(sizes), 2)).astype(np.int32)
    return F, C


@pytest.mark.parametrize("seed", range(6))
def test_retrieve_equals_python_loops(seed):
    rng = np.random.default_rng(10 + seed)
    n_sub = int(rng.integers(1, 5))
    sizes = [int(x) for x in rng.integers(1, 120, n_sub)]
    F, C = _tiny_db(rng, n_sub, sizes)
    B, M, N = 3, int(rng.choice([1, 3, 5])), int(rng.choice([1, 5, 15, 17]))
    Q = F[rng.integers(0, F.shape[0], B * M)].reshape(B, M, 64).copy()
    Q[0, 0] += np.float32(1e-3)
    cand = oracle.retrieve(sizes, F, C, Q, N)
    off = np.concatenate([[0], np.cumsum(sizes)])
    w = 0
    for b in range(B):
        for j in range(M):
            for i in range(n_sub):
                Fi = F[off[i]:off[i + 1]]
                acc = np.array([oracle.acc(Q[b, j], f) for f in Fi], np.float32)
                exp = _python_topn(acc, N)
                c = len(exp)
                assert np.all(cand.subspace[w:w + c] == i)
                assert np.all(cand.bundle[w:w + c] == b) and np.all(cand.qframe[w:w + c] == j)
                assert np.array_equal(cand.frame[w:w + c], exp)
                assert np.array_equal(cand.acc[w:w + c], acc[exp])
                assert np.array_equal(cand.dist[w:w + c], np.sqrt(acc[exp]))
                assert np.array_equal(cand.x[w:w + c], C[off[i] + exp, 0])
                assert np.array_equal(cand.y[w:w + c], C[off[i] + exp, 1])
                w += c
    assert w == len(cand) == B * M * sum(min(N, s) for s in sizes)


def test_select_path_equals_sortall_path():
    rng = np.random.default_rng(99)
    sizes = [300, 7, 50]
    F, C = _tiny_db(rng, 3, sizes)
    Q = F[[0, 5, 310, 200]].reshape(2, 2, 64)
    a = oracle.retrieve(sizes, F, C, Q, 15, use_select=False)
    b = oracle.retrieve(sizes, F, C, Q, 15, use_select=True)
    for k in a.__dataclass_fields__:
        assert np.array_equal(getattr(a, k), getattr(b, k))


def test_self_query_first_at_zero_and_duplicates_adjacent():
    rng = np.random.default_rng(1)
    F, C = _tiny_db(rng, 1, [200])
    cand = oracle.retrieve([200], F, C, F[1][None, None, :], 5)
    assert cand.acc[0] == 0.0 and cand.frame[0] == 1
    # F[3] and F[199] are copies of F[1]: all three tie at +0, by index
    assert list(cand.frame[:3]) == [1, 3, 199] and np.all(cand.acc[:3] == 0.0)
    assert np.all(np.diff(cand.acc) >= 0)


def test_undersized_subspace():
    rng = np.random.default_rng(2)
    F, C = _tiny_db(rng, 2, [7, 40], dup=False)
    cand = oracle.retrieve([7, 40], F, C, F[0][None, None, :], 15)
    assert len(cand) == 7 + 15 and np.array_equal(np.sort(cand.frame[:7]), np.arange(7))


def test_paper_825_candidates():
    g = json.load(open(os.path.join(GOLD, "paper_constants.json")))
    N, M, P = g["N"]["value"], g["M"]["value"], g["P"]["value"]
    spec = synthgen.Spec(seed=2, n_floors=1, paths=P, frames_per_path=60)
    F, C = synthgen.db_host(spec)
    video = synthgen.render_host(spec, synthgen.query_points(spec, 5, 40, "path", 0, 2))["desc"]
    first, ln = oracle.select_window(40, 20, M)
    cand = oracle.retrieve([60] * P, F, C, video[first:first + ln][None], N)
    assert len(cand) == N * M * P == g["candidates"]["value"]


def test_select_window_spec_examples():
    for ex in json.load(open(os.path.join(GOLD, "spec_examples.json")))["window"]:
        first, ln = oracle.select_window(ex["n_frames"], ex["m"], ex["M"])
        assert list(range(first, first + ln)) == ex["frames"], ex
    with pytest.raises(ValueError):
        oracle.select_window(20, 3, 4)     # M even
    with pytest.raises(ValueError):
        oracle.select_window(20, 20, 3)    # m out of range


def test_select_window_properties():
    # length min(M, L), contains m, centred on m when the centred window fits,
    # otherwise flush against the sequence end it would overrun
    for L in range(1, 15):
        for M in (1, 3, 5, 11, 13):
            h = (M - 1) // 2
            for m in range(L):
                first, ln = oracle.select_window(L, m, M)
                assert ln == min(M, L) and 0 <= first and first + ln <= L
                assert first <= m < first + ln
                if m - h >= 0 and m + h < L:
                    assert first == m - h
                elif m - h < 0:
                    assert first == 0
                else:
                    assert first + ln == L
