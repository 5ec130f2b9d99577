"""NEXT-4 host logic of the localisation service: NDJSON framing,
protocol totality (one response per line, errors included), request-order
responses per connection, request validation, micro-batching by (M, params), and the
streaming window (P:149 selectNearbyFrames via ol_select_window).  The retrieval
itself is replaced by a recording stub here (no GPU on this host); the GPU test
(test_gpu_service.py) runs the real engine against the oracle."""
import json
import threading

import numpy as np
import pytest

import paper_2006_08861_b200 as ol
from paper_2006_08861_b200 import service


class StubEngine:
    """Records every query; the 'estimate' of a bundle encodes its shape and first value."""

    def __init__(self):
        self.params = ol.Params()
        self.calls = []
        self._last = None
        self.lock = threading.Lock()

    def query(self, frames, params=None, aggregate=True):
        with self.lock:
            self.calls.append((frames.shape, params))
            self._last = frames.copy()

    def estimates(self):
        f = self._last
        out = np.zeros(f.shape[0], ol.ESTIMATE_DTYPE)
        out["x"] = f.shape[1]                    # M
        out["y"] = np.round(f[:, 0, 0] * 1000)   # identifies the bundle
        out["confidence"] = 0.5
        out["total"] = f.shape[1] * 15
        out["n_ranked"] = 1
        out["ranked"][:, 0]["count"] = 7
        return out


@pytest.fixture
def svc():
    s = service.LocService(StubEngine(), stream_M=5, batch_window_s=0.002)
    yield s
    s.close()


def _bundle(M, v=0.1):
    b = np.full((M, 64), 0.01, np.float64)
    b[0, 0] = v
    return b.tolist()


def test_valid_bundle(svc):
    r = svc.handle_line(json.dumps({"id": 7, "features": _bundle(3, 0.25)}))
    assert r["id"] == 7 and r["x"] == 3 and r["y"] == 250 and r["ranked_tiles"] == [[0, 0, 7, 0]]
    assert r["timing_ms"] >= 0 and "error" not in r


@pytest.mark.parametrize("line,code", [
    ("{not json", "parse_error"),
    ("[1, 2]", "parse_error"),
    (json.dumps({"id": 1}), "parse_error"),
    (json.dumps({"id": 1, "features": [[0.0] * 63]}), "dimension_mismatch"),
    (json.dumps({"id": 1, "features": [0.0] * 64}), "dimension_mismatch"),
    (json.dumps({"id": 1, "features": _bundle(2)}), "invalid_argument"),             # M even
    (json.dumps({"id": 1, "features": _bundle(65)}), "invalid_argument"),            # M > 64
    (json.dumps({"id": 1, "features": [["a"] * 64]}), "parse_error"),
    (json.dumps({"id": 1, "features": _bundle(1), "params": {"N": 0}}), "invalid_argument"),
    (json.dumps({"id": 1, "features": _bundle(1), "params": {"toler_per": 1.5}}), "invalid_argument"),
    (json.dumps({"id": 1, "features": _bundle(1), "params": {"top_c": 2.5}}), "invalid_argument"),
])
def test_errors_are_single_responses(svc, line, code):
    r = svc.handle_line(line)
    assert r["error"] == code and "message" in r


def test_nonfinite_rejected(svc):
    b = _bundle(1)
    line = json.dumps({"id": 3, "features": b}).replace("0.01", "NaN", 1)
    assert svc.handle_line(line)["error"] == "nonfinite"


def test_tcp_order_totality_and_batching(svc):
    srv, addr = service.serve(svc)
    try:
        reqs = []
        for i in range(40):
            if i % 7 == 3:
                reqs.append("{broken")
            else:
                reqs.append({"id": i, "features": _bundle(1 + 2 * (i % 3), 0.001 * i)})
        outs = {}

        def client(k):
            outs[k] = service.request(addr, reqs)

        th = [threading.Thread(target=client, args=(k,)) for k in range(4)]
        [t.start() for t in th]
        [t.join() for t in th]
        for k in range(4):
            rs = outs[k]
            assert len(rs) == len(reqs)                      # one response per line
            for q, r in zip(reqs, rs):                       # in request order
                if isinstance(q, str):
                    assert r["error"] == "parse_error"
                else:
                    assert r["id"] == q["id"] and r["x"] == len(q["features"])
                    assert r["y"] == round(q["features"][0][0] * 1000)
        # every engine call holds bundles of a single M (grouped micro-batches)
        for shape, _ in svc.engine.calls:
            assert len(shape) == 3 and shape[2] == 64
        assert svc.batches <= 4 * 40
    finally:
        srv.shutdown()


def test_stream_window_is_select_window(svc):
    # M = 5 centred window on the newest frame, clamped: sizes 1, 1 (2 -> drop
    # the oldest to keep M odd), 3, 3, 5, 5, ...
    sizes = []
    for t in range(8):
        r = svc.handle_line(json.dumps({"id": t, "user": "u1", "feature": [0.01 * (t + 1)] + [0.0] * 63}))
        sizes.append(r["x"])
        assert r["y"] == round(0.01 * (t + 1 - (r["x"] - 1)) * 1000)   # the window ends at frame t
    assert sizes == [1, 1, 3, 3, 5, 5, 5, 5]
    # users do not share history
    r = svc.handle_line(json.dumps({"id": 99, "user": "u2", "feature": [0.5] + [0.0] * 63}))
    assert r["x"] == 1 and r["y"] == 500
