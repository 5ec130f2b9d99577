"""Shared helpers for the -m gpu parity tests (compare product vs oracle)."""
import numpy as np

import oracle


def assert_candidates_equal(got: np.ndarray, ref: "oracle.Candidates", ctx=""):
    assert len(got) == len(ref), f"{ctx}: {len(got)} vs {len(ref)} candidates"
    for gk, rk in (("subspace", "subspace"), ("frame", "frame"), ("bundle", "bundle"),
                   ("query_frame", "qframe"), ("x", "x"), ("y", "y")):
        g, r = got[gk], getattr(ref, rk)
        if not np.array_equal(g, r):
            i = int(np.nonzero(g != r)[0][0])
            raise AssertionError(f"{ctx}: field {gk} differs first at {i}: {g[i]} vs {r[i]} "
                                 f"(frame {got['frame'][i]} vs {ref.frame[i]}, acc {got['dist2'][i]!r} vs {ref.acc[i]!r})")
    assert np.array_equal(got["dist2"].view(np.uint32), ref.acc.view(np.uint32)), ctx
    assert np.array_equal(got["dist"].view(np.uint32), ref.dist.view(np.uint32)), ctx


def assert_estimates_equal(est: np.ndarray, ref: "oracle.Candidates", params=None, ctx=""):
    params = params or {}
    for b in range(est.shape[0]):
        sel = ref.bundle == b
        e = oracle.aggregate(np.column_stack([ref.x[sel], ref.y[sel]]), **params)
        g = est[b]
        assert (int(g["x"]), int(g["y"]), bool(g["low_confidence"])) == (e.x, e.y, e.low_confidence), \
            f"{ctx} bundle {b}: {(g['x'], g['y'], g['low_confidence'])} vs {(e.x, e.y, e.low_confidence)}"
        assert g["confidence"] == e.confidence, ctx
        assert g["x_m"] == e.x_m and g["y_m"] == e.y_m, f"{ctx} bundle {b}: metres"
        k = int(g["n_ranked"])
        assert k == len(e.ranked_count)
        assert np.array_equal(g["ranked"]["x"][:k], e.ranked_xy[:, 0])
        assert np.array_equal(g["ranked"]["y"][:k], e.ranked_xy[:, 1])
        assert np.array_equal(g["ranked"]["count"][:k], e.ranked_count)
        assert np.array_equal(g["ranked"]["circle"][:k], e.ranked_circle)
        assert int(g["total"]) == int(sel.sum())
