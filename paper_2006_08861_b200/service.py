"""Localisation service front end (NEXT-4 in SURVEY §8f): the paper's client/server
split (Fig. 2, "Parallel retrieving with GPU in the remote server";
P:139 the client sends each frame's feature).  Newline-delimited JSON over TCP
(S:319-370): one request object per line, exactly one response object per line,
responses on a connection in request order, malformed requests answered with an
error object while the connection stays usable.

Requests
  {"id": any, "features": [[64 floats] x M]}            a bundle (M odd, 1..64)
  {"id": any, "user": key, "feature": [64 floats]}      streaming: appended to the
      user's history; answered for the newest frame with the window of
      ol_select_window (P:149 selectNearbyFrames, clamped, M = the service's M)
  optional "params": {"N", "top_c", "toler_per", "radius_m"} overrides
Responses
  {"id", "x", "y", "x_m", "y_m", "confidence", "low_confidence", "total",
   "ranked_tiles": [[x, y, count, circle], ...], "timing_ms"}
  {"id", "error": code, "message"}   code in parse_error, dimension_mismatch,
      invalid_argument, nonfinite, internal

All retrieval and aggregation run in the CUDA library through ``Engine.query``;
requests that arrive together are micro-batched into one query per (M, params)
group (results are independent of batching: every bundle is scored alone).
"""
from __future__ import annotations

import json
import math
import queue
import socket
import socketserver
import threading
import time
from collections import defaultdict, deque
from dataclasses import dataclass, field

import numpy as np

from . import Params, select_window, OmnilocError

K = 64


class RequestError(Exception):
    def __init__(self, code: str, message: str):
        super().__init__(message)
        self.code = code


def _floats(v, what):
    try:
        a = np.asarray(v, dtype=np.float64)
    except (TypeError, ValueError):
        raise RequestError("parse_error", f"{what} must be numbers")
    if a.dtype == object:
        raise RequestError("parse_error", f"{what} must be numbers")
    return a


def parse_params(base: Params, d) -> Params:
    if d is None:
        return base
    if not isinstance(d, dict):
        raise RequestError("parse_error", "params must be an object")
    p = Params(base.N, base.top_c, base.toler_per, base.radius_m, base.tile_m)
    for k in ("N", "top_c"):
        if k in d:
            v = d[k]
            if not isinstance(v, int) or isinstance(v, bool):
                raise RequestError("invalid_argument", f"{k} must be an integer")
            setattr(p, k, v)
    for k in ("toler_per", "radius_m"):
        if k in d:
            v = d[k]
            if not isinstance(v, (int, float)) or isinstance(v, bool) or not math.isfinite(v):
                raise RequestError("invalid_argument", f"{k} must be a finite number")
            setattr(p, k, float(v))
    if not (1 <= p.N <= 128) or not (1 <= p.top_c <= 64) or not (0 < p.toler_per <= 1) or not (p.radius_m > 0):
        raise RequestError("invalid_argument", "params outside N 1..128, top_c 1..64, toler_per (0,1], radius_m > 0")
    return p


def bundle_from(features) -> np.ndarray:
    """[M][64] fp32 bundle from the wire (1 <= M <= 64, M odd, length K each)."""
    a = _floats(features, "features")
    if a.ndim != 2:
        raise RequestError("dimension_mismatch", "features must be an array of M arrays")
    M, k = a.shape
    if k != K:
        raise RequestError("dimension_mismatch", f"each feature must have {K} values, got {k}")
    if M < 1 or M > 64 or M % 2 == 0:
        raise RequestError("invalid_argument", f"M = {M}: must be odd, 1..64 (P:139 centred window)")
    if not np.all(np.isfinite(a)):
        raise RequestError("nonfinite", "feature values must be finite (S:32)")
    return a.astype(np.float32)


@dataclass
class _Job:
    req_id: object
    bundle: np.ndarray
    params: Params
    t0: float
    done: threading.Event = field(default_factory=threading.Event)
    response: dict | None = None


class LocService:
    """Owns an uploaded Engine; one worker thread micro-batches pending bundles."""

    def __init__(self, engine, params: Params | None = None, stream_M: int = 5,
                 batch_window_s: float = 0.0005, max_batch: int = 256):
        self.engine = engine
        self.params = params or engine.params
        self.stream_M = stream_M
        self.batch_window_s = batch_window_s
        self.max_batch = max_batch
        self._q: queue.Queue = queue.Queue()
        self._hist = defaultdict(lambda: deque(maxlen=64))
        self._hist_lock = threading.Lock()
        self._stop = threading.Event()
        self._worker = threading.Thread(target=self._run, daemon=True)
        self._worker.start()
        self.batches = 0

    # ---------------------------------------------------------------- requests
    def handle_line(self, line: bytes | str) -> dict:
        """One request line -> one response object (never raises)."""
        t0 = time.perf_counter()
        rid = None
        try:
            try:
                req = json.loads(line)
            except (ValueError, UnicodeDecodeError) as e:
                raise RequestError("parse_error", f"malformed JSON: {e}")
            if not isinstance(req, dict):
                raise RequestError("parse_error", "request must be a JSON object")
            rid = req.get("id")
            params = parse_params(self.params, req.get("params"))
            if "features" in req:
                bundle = bundle_from(req["features"])
            elif "feature" in req and "user" in req:
                f = bundle_from([req["feature"]])[0]
                with self._hist_lock:
                    h = self._hist[json.dumps(req["user"], sort_keys=True)]
                    h.append(f)
                    frames = list(h)
                first, ln = select_window(len(frames), len(frames) - 1, self.stream_M)
                bundle = np.stack(frames[first:first + ln])
                if bundle.shape[0] % 2 == 0:   # history shorter than M and even: drop the oldest
                    bundle = bundle[1:]
            else:
                raise RequestError("parse_error", "request needs 'features' or 'user' + 'feature'")
            job = _Job(rid, bundle, params, t0)
            self._q.put(job)
            job.done.wait()
            return job.response
        except RequestError as e:
            return {"id": rid, "error": e.code, "message": str(e)}
        except Exception as e:  # protocol totality: every line gets exactly one response
            return {"id": rid, "error": "internal", "message": str(e)}

    # ---------------------------------------------------------------- worker
    def _run(self):
        while not self._stop.is_set():
            try:
                first = self._q.get(timeout=0.1)
            except queue.Empty:
                continue
            jobs = [first]
            deadline = time.perf_counter() + self.batch_window_s
            while len(jobs) < self.max_batch:
                try:
                    jobs.append(self._q.get(timeout=max(0.0, deadline - time.perf_counter())))
                except queue.Empty:
                    break
            groups = defaultdict(list)
            for j in jobs:
                p = j.params
                groups[(j.bundle.shape[0], p.N, p.top_c, p.toler_per, p.radius_m, p.tile_m)].append(j)
            for (M, *_), js in groups.items():
                self._answer(M, js)

    def _answer(self, M, js):
        try:
            frames = np.ascontiguousarray(np.stack([j.bundle for j in js]))   # [B][M][64]
            self.engine.query(frames, params=js[0].params, aggregate=True)
            est = self.engine.estimates()
            self.batches += 1
            for j, e in zip(js, est):
                n = int(e["n_ranked"])
                j.response = {"id": j.req_id, "x": int(e["x"]), "y": int(e["y"]),
                              "x_m": float(e["x_m"]), "y_m": float(e["y_m"]),
                              "confidence": float(e["confidence"]),
                              "low_confidence": bool(e["low_confidence"]), "total": int(e["total"]),
                              "ranked_tiles": [[int(r["x"]), int(r["y"]), int(r["count"]), int(r["circle"])]
                                               for r in e["ranked"][:n]],
                              "timing_ms": (time.perf_counter() - j.t0) * 1e3}
        except OmnilocError as err:
            code = {"NONFINITE": "nonfinite", "INVALID_ARGUMENT": "invalid_argument",
                    "DIMENSION_MISMATCH": "dimension_mismatch"}.get(str(err).split(":")[0][7:], "internal")
            for j in js:
                j.response = {"id": j.req_id, "error": code, "message": str(err)}
        except Exception as err:
            for j in js:
                j.response = {"id": j.req_id, "error": "internal", "message": str(err)}
        for j in js:
            j.done.set()

    def close(self):
        self._stop.set()
        self._worker.join(timeout=2)


class _Handler(socketserver.StreamRequestHandler):
    def handle(self):
        svc: LocService = self.server.svc
        for line in self.rfile:
            if not line.strip():
                continue
            resp = svc.handle_line(line)
            self.wfile.write((json.dumps(resp) + "\n").encode())
            self.wfile.flush()


class _Server(socketserver.ThreadingMixIn, socketserver.TCPServer):
    daemon_threads = True
    allow_reuse_address = True


def serve(svc: LocService, host: str = "127.0.0.1", port: int = 0):
    """Start the TCP front end on a background thread; returns (server, (host, port))."""
    srv = _Server((host, port), _Handler)
    srv.svc = svc
    threading.Thread(target=srv.serve_forever, daemon=True).start()
    return srv, srv.server_address


def request(addr, objs, timeout: float = 30.0):
    """Tiny client: send request objects on one connection, return the responses."""
    with socket.create_connection(addr, timeout=timeout) as s:
        f = s.makefile("rwb")
        for o in objs:
            f.write(((o if isinstance(o, str) else json.dumps(o)) + "\n").encode())
        f.flush()
        return [json.loads(f.readline()) for _ in objs]


def main(argv=None):
    """python -m paper_2006_08861_b200.service --db features.npy coords.npy sizes.npy --grid W H
    [--bind 127.0.0.1:7700] [--M 5]: serve a database of fp32 descriptors [n][64], int32 tiles
    [n][2] and subspace sizes (S:341 serve --db DB --bind ADDR)."""
    import argparse
    ap = argparse.ArgumentParser(prog="paper_2006_08861_b200.service")
    ap.add_argument("--db", nargs=3, required=True, metavar=("FEATURES", "COORDS", "SIZES"))
    ap.add_argument("--grid", nargs=2, type=int, required=True)
    ap.add_argument("--bind", default="127.0.0.1:7700")
    ap.add_argument("--M", type=int, default=5)
    a = ap.parse_args(argv)
    from . import Engine
    try:
        F = np.load(a.db[0]).astype(np.float32)
        C = np.load(a.db[1]).astype(np.int32)
        sizes = [int(s) for s in np.load(a.db[2])]
        eng = Engine(0)
        eng.upload(F, C, sizes, tuple(a.grid))
    except Exception as e:   # DB load failure: its own exit code
        print(f"database load failed: {e}")
        raise SystemExit(3)
    host, port = a.bind.rsplit(":", 1)
    try:
        srv, addr = serve(LocService(eng, stream_M=a.M), host, int(port))
    except OSError as e:     # bind failure
        print(f"bind failed: {e}")
        raise SystemExit(4)
    print(f"serving on {addr[0]}:{addr[1]}", flush=True)
    threading.Event().wait()


if __name__ == "__main__":
    main()
