"""Pins for the oracle's Algorithm 2 -- CPU only.

External pins: hand-constructed cases from SPEC,
the circle-boundary geometry (tile offsets (6,8) in / (7,8) out at 3 m / 0.3 m),
the 165/825 vs 166/825 threshold, invariances, and an independent
Python implementation that bins on a dense numpy grid and computes the circle
count of EVERY tile by a 2-D window sum ("exhaustive all-tiles").
"""
import json
import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def dense_reference(xy, top_c=10, toler_per=0.2, radius_m=3.0, tile_m=0.3):
    xy = np.asarray(xy, np.int64).reshape(-1, 2)
    R = int(np.floor(radius_m / tile_m)) + 1
    x0, y0 = xy.min(0) - R
    x1, y1 = xy.max(0) + R
    grid = np.zeros((y1 - y0 + 1, x1 - x0 + 1), np.int64)
    np.add.at(grid, (xy[:, 1] - y0, xy[:, 0] - x0), 1)
    r2 = (radius_m / tile_m) ** 2
    offs = [(dx, dy) for dx in range(-R, R + 1) for dy in range(-R, R + 1)
            if float(dx * dx + dy * dy) <= r2]
    circ = np.zeros_like(grid)
    H, W = grid.shape
    for dx, dy in offs:    # circle(t) = sum of counts at t + (dx, dy)
        src = grid[max(dy, 0):H + min(dy, 0), max(dx, 0):W + min(dx, 0)]
        circ[max(-dy, 0):H + min(-dy, 0), max(-dx, 0):W + min(-dx, 0)] += src
    ys, xs = np.nonzero(grid)
    tiles = sorted(zip(-grid[ys, xs], ys + y0, xs + x0))[:top_c]
    ranked = [(int(x), int(y), int(-c), int(circ[y - y0, x - x0])) for c, y, x in tiles]
    total = xy.shape[0]
    for x, y, c, ci in ranked:
        if ci > toler_per * total:
            return (x, y, ci / total, False, ranked)
    best = max(range(len(ranked)), key=lambda i: (ranked[i][3], -i))
    x, y, c, ci = ranked[best]
    return (x, y, ci / total, True, ranked)


def _check(xy, **kw):
    e = oracle.aggregate(xy, **kw)
    x, y, conf, low, ranked = dense_reference(xy, **kw)
    assert (e.x, e.y, e.low_confidence) == (x, y, low)
    assert e.confidence == conf
    assert [tuple(v) for v in np.column_stack([e.ranked_xy, e.ranked_count, e.ranked_circle])] \
        == ranked
    return e


def test_point_mass():
    g = json.load(open(os.path.join(GOLD, "spec_examples.json")))["point_mass"]
    e = _check([g["tile"]] * g["count"])
    assert (e.x, e.y) == tuple(g["tile"]) and e.confidence == 1.0 and not e.low_confidence
    assert e.ranked_count[0] == g["count"] and e.ranked_circle[0] == g["count"]


def test_empty_is_error():
    with pytest.raises(LookupError):
        oracle.aggregate(np.zeros((0, 2), np.int32))


def test_rank_tie_break():
    g = json.load(open(os.path.join(GOLD, "spec_examples.json")))["rank_tie"]
    far = [[100, 100]]
    e = oracle.aggregate(g["tiles"] + far, top_c=10)
    assert tuple(e.ranked_xy[0]) == tuple(g["first"])


def test_circle_boundary_geometry():
    # radius 3 m / 0.3 m tiles = 10 tiles, inclusive: (6,8),(8,6),(10,0),(7,7) in; (7,8) out
    base = [[50, 50]] * 3
    for off, inside in [((6, 8), True), ((8, 6), True), ((10, 0), True), ((0, 10), True),
                        ((7, 7), True), ((7, 8), False), ((11, 0), False)]:
        e = oracle.aggregate(base + [[50 + off[0], 50 + off[1]]], toler_per=0.99)
        assert e.ranked_circle[0] == 3 + int(inside), off


def test_threshold_strict_165_vs_166():                  # P:187 ">" ; 0.2 * 825 = 165
    far = [[1000 + 30 * i, 1000] for i in range(825)]
    for k, passes in ((165, False), (166, True)):
        xy = [[10, 10]] * k + far[: 825 - k]
        e = _check(xy)
        assert (not e.low_confidence) == passes and (e.x, e.y) == (10, 10)


def test_spike_vs_cluster():
    total = 1000
    spike = [[10, 10]] * 150                              # A: 15 %, isolated
    cluster = [[100, 100]] * 100                          # B itself: 10 %
    rng = np.random.default_rng(0)
    ring = []
    while len(ring) < 500:                                # 50 % more within 3 m of B
        dx, dy = rng.integers(-9, 10, 2)
        if 0 < dx * dx + dy * dy <= 81 and (dx, dy) != (0, 0):
            ring.append([100 + dx, 100 + dy])
    noise = [[400 + 25 * i, 400 + 25 * (i % 7)] for i in range(total - 750)]
    e = _check(spike + cluster + ring + noise)
    assert tuple(e.ranked_xy[0]) == (10, 10)              # A ranks first ...
    assert (e.x, e.y) == (100, 100) and not e.low_confidence   # ... but B wins
    assert e.confidence >= 0.6


def test_uniform_scatter_falls_back():
    xy = [[25 * i, 25 * j] for i in range(20) for j in range(20)]
    e = _check(xy)
    assert e.low_confidence


@pytest.mark.parametrize("seed", range(200))
def test_random_sets_vs_dense_exhaustive(seed):
    rng = np.random.default_rng(seed)
    kind = seed % 4
    n = int(rng.integers(1, 900))
    if kind == 0:
        xy = rng.integers(0, 40, (n, 2))
    elif kind == 1:
        c = rng.integers(0, 300, (5, 2))
        xy = c[rng.integers(0, 5, n)] + rng.integers(-6, 7, (n, 2))
    elif kind == 2:
        xy = rng.integers(0, 2000, (n, 2))
    else:
        xy = np.concatenate([rng.integers(0, 10, (n // 2 + 1, 2)), rng.integers(0, 500, (n // 2, 2))])
    kw = dict(top_c=int(rng.choice([1, 3, 10, 64])), toler_per=float(rng.choice([0.2, 0.05, 0.5, 1.0])),
              radius_m=float(rng.choice([3.0, 1.5, 0.9])), tile_m=0.3)
    _check(np.abs(xy).astype(np.int32), **kw)


def test_invariances():
    rng = np.random.default_rng(5)
    for _ in range(30):
        xy = rng.integers(0, 60, (int(rng.integers(5, 300)), 2)).astype(np.int32)
        e = oracle.aggregate(xy)
        assert np.all(e.ranked_circle <= len(xy))                           # conservation
        p = oracle.aggregate(xy[rng.permutation(len(xy))])                 # permutation
        assert (p.x, p.y, p.confidence, p.low_confidence) == (e.x, e.y, e.confidence, e.low_confidence)
        d = rng.integers(0, 1000, 2).astype(np.int32)
        t = oracle.aggregate(xy + d)                                        # translation
        assert (t.x - d[0], t.y - d[1], t.confidence, t.low_confidence) == \
            (e.x, e.y, e.confidence, e.low_confidence)


def test_majority_guarantee():
    rng = np.random.default_rng(6)
    for _ in range(20):
        n = 500
        k = int(n * 0.2) + 1 + int(rng.integers(0, 200))
        xy = np.concatenate([np.full((k, 2), 77), rng.integers(200, 900, (n - k, 2))]).astype(np.int32)
        e = oracle.aggregate(xy)
        assert (e.x, e.y) == (77, 77) and not e.low_confidence


def test_metres_are_correctly_rounded_tile_centres():        # S:329, DESIGN R14
    """x_m = tile_m * x is the binary64 product, i.e. the exact rational product of the
    binary64 tile_m and the tile index, rounded once to nearest (Fraction -> float rounds
    correctly); checked for positive, negative and large tiles and a non-default tile_m."""
    from fractions import Fraction
    for tile_m in (0.3, 0.25, 0.1):
        for t in ((10, 20), (-7, 3), (123456, -654321), (0, 0)):
            e = oracle.aggregate(np.array([t], np.int32), tile_m=tile_m, radius_m=3 * tile_m / 0.3)
            assert (e.x, e.y) == t
            assert e.x_m == float(Fraction(tile_m) * t[0])
            assert e.y_m == float(Fraction(tile_m) * t[1])
    # the tile centre is not the decimal product when tile_m is not a dyadic rational
    e = oracle.aggregate(np.array([[3, 0]], np.int32))
    assert e.x_m != 0.9 and abs(e.x_m - 0.9) <= np.spacing(0.9)
