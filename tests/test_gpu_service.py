"""NEXT-4 on the GPU: the localisation service answers every request
exactly like the offline path -- Alg. 1 retrieval + Alg. 2 aggregation computed by the
oracle on the same bundle (S:353 service/CLI equivalence; JSON floats round-trip
exactly), under concurrent clients (request isolation), including streaming users."""
import json
import threading

import numpy as np
import pytest

import oracle
import synthgen
import paper_2006_08861_b200 as ol
from paper_2006_08861_b200 import service

pytestmark = pytest.mark.gpu


def _offline(F, C, sizes, bundle, N=15):
    ref = oracle.retrieve(sizes, F, C, bundle[None], N)
    return oracle.aggregate(np.column_stack([ref.x, ref.y]))


def test_service_matches_offline_path_under_concurrency():
    spec = synthgen.Spec(seed=61, n_floors=1, paths=5, frames_per_path=600)   # C2-shaped: 5 path subspaces
    F, C = synthgen.db_host(spec)
    sizes = [600] * 5
    eng = ol.Engine(0)
    eng.upload(F, C, sizes, spec.grid())
    svc = service.LocService(eng, stream_M=5)
    srv, addr = service.serve(svc)
    try:
        video = synthgen.render_host(spec, synthgen.query_points(spec, 5, 40, "path", 0, 2))["desc"]
        rng = np.random.default_rng(0)
        reqs = []
        for i in range(30):
            M = int(rng.choice([1, 3, 5, 11]))
            m = int(rng.integers(0, 40))
            first, ln = ol.select_window(40, m, M)
            reqs.append({"id": i, "features": video[first:first + ln].tolist()})
        reqs.append({"id": "bad", "features": [[0.0] * 63]})
        outs = {}

        def client(k):
            outs[k] = service.request(addr, reqs)

        th = [threading.Thread(target=client, args=(k,)) for k in range(6)]
        [t.start() for t in th]
        [t.join() for t in th]
        for k in range(6):
            for q, r in zip(reqs, outs[k]):
                if q["id"] == "bad":
                    assert r["error"] == "dimension_mismatch"
                    continue
                e = _offline(F, C, sizes, np.asarray(q["features"], np.float32))
                assert (r["x"], r["y"], r["low_confidence"]) == (e.x, e.y, e.low_confidence), q["id"]
                assert r["confidence"] == e.confidence
                assert r["x_m"] == 0.3 * e.x and r["y_m"] == 0.3 * e.y
                assert [t[:3] for t in r["ranked_tiles"]] == [[int(a), int(b), int(c)] for (a, b), c in
                                                               zip(e.ranked_xy, e.ranked_count)]
        # streaming user: frame t is answered with the clamped centred window ending at t
        for t in range(7):
            r = svc.handle_line(json.dumps({"id": t, "user": "walker", "feature": video[t].tolist()}))
            first, ln = ol.select_window(t + 1, t, 5)
            win = video[first:first + ln]
            if win.shape[0] % 2 == 0:
                win = win[1:]
            e = _offline(F, C, sizes, win)
            assert (r["x"], r["y"], r["confidence"]) == (e.x, e.y, e.confidence)
    finally:
        srv.shutdown()
        svc.close()
