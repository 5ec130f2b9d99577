"""Plain CPU ORACLE for arXiv 2006.08861's hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` leg may import this package.  The product package
(``paper_2006_08861_b200``) never imports it and shares no code with it.

The arithmetic lives in ``oracle.c`` (plain C, ``-ffp-contract=off``); this
module only builds it with gcc and marshals numpy arrays.  See the header of
``oracle.c`` for the citations and DESIGN.md §3 for the readings it follows.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

OR_OK, OR_ERR_INVALID, OR_ERR_EMPTY, OR_ERR_RANGE, OR_ERR_CAPACITY = 0, -1, -2, -3, -4


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so (gcc, -O2, no contraction, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call([
            "gcc", "-O2", "-std=c11", "-D_GNU_SOURCE", "-ffp-contract=off", "-fno-fast-math",
            "-fopenmp", "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P = ctypes.c_void_p
        i64, i32, u32, dbl, flt = (ctypes.c_int64, ctypes.c_int, ctypes.c_uint32,
                                   ctypes.c_double, ctypes.c_float)
        L.oracle_extract_feature.argtypes = [P, i32, i32, P, P]
        L.oracle_extract_feature.restype = i32
        L.oracle_acc.argtypes = [P, P, i32]
        L.oracle_acc.restype = flt
        L.oracle_distance.argtypes = [P, P, i32]
        L.oracle_distance.restype = flt
        L.oracle_acc_many.argtypes = [P, P, i64, i32, P]
        L.oracle_acc_many.restype = None
        L.oracle_topn_sortall.argtypes = [P, i64, i32, P, P]
        L.oracle_topn_sortall.restype = i64
        L.oracle_topn_select.argtypes = [P, i64, i32, P, P]
        L.oracle_topn_select.restype = i64
        L.oracle_select_window.argtypes = [u32, u32, u32, P, P]
        L.oracle_select_window.restype = i32
        L.oracle_retrieve.argtypes = [i32, P, P, P, i32, i32, i32, P, i32, i32,
                                      P, P, P, P, P, P, P, P, i64]
        L.oracle_retrieve.restype = i64
        L.oracle_aggregate.argtypes = [i64, P, i32, dbl, dbl, dbl, P, P, P, P, P, P, P, P]
        L.oracle_aggregate.restype = i32
        L.oracle_shift_distance.argtypes = [P, P, i32, P]
        L.oracle_shift_distance.restype = flt
        L.oracle_shift_profile.argtypes = [P, i32, i32, P, P]
        L.oracle_shift_profile.restype = i32
        L.oracle_set_threads.argtypes = [i32]
        L.oracle_set_threads.restype = None
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


# --------------------------------------------------------------------------- feature
def extract_feature(profile, K: int = 64):
    """|DFT| bins 1..K of a circular profile, L2-normalised."""
    p = _c(profile, np.float64)
    out = np.zeros(K, np.float64)
    deg = ctypes.c_int(0)
    rc = lib().oracle_extract_feature(_p(p), p.shape[0], K, _p(out), ctypes.byref(deg))
    if rc != OR_OK:
        raise ValueError(f"oracle_extract_feature rc={rc}")
    return out, bool(deg.value)


def set_threads(n: int):
    """OpenMP threads of the oracle's parallel loops (timing only; n < 1: all cores)."""
    lib().oracle_set_threads(int(n))


def shift_profile(profile, K: int = 64):
    """NEXT-1 stored profile: (x - mean x) / ||m||, ||m|| the descriptor's normaliser
    (|DFT| bins 1..K) -> (binary64 [W], fp32 [W] = RN32 of it); zeros if degenerate."""
    p = _c(profile, np.float64)
    o64 = np.zeros(p.shape[0], np.float64)
    o32 = np.zeros(p.shape[0], np.float32)
    rc = lib().oracle_shift_profile(_p(p), p.shape[0], K, _p(o64), _p(o32))
    if rc != OR_OK:
        raise ValueError(f"oracle_shift_profile rc={rc}")
    return o64, o32


# --------------------------------------------------------------------------- distance
def acc(q, f) -> np.float32:
    """fp32 fixed-order squared distance (DESIGN R3)."""
    q = _c(q, np.float32); f = _c(f, np.float32)
    return np.float32(lib().oracle_acc(_p(q), _p(f), q.shape[0]))


def distance(q, f) -> np.float32:
    q = _c(q, np.float32); f = _c(f, np.float32)
    return np.float32(lib().oracle_distance(_p(q), _p(f), q.shape[0]))


def acc_many(q, F) -> np.ndarray:
    q = _c(q, np.float32); F = _c(F, np.float32)
    out = np.empty(F.shape[0], np.float32)
    lib().oracle_acc_many(_p(q), _p(F), F.shape[0], F.shape[1], _p(out))
    return out


def topn(acc_arr, N: int, method: str = "sortall"):
    """N smallest of (acc, index), ascending. -> (idx u32, acc f32)."""
    a = _c(acc_arr, np.float32)
    idx = np.zeros(N, np.uint32); ta = np.zeros(N, np.float32)
    fn = lib().oracle_topn_sortall if method == "sortall" else lib().oracle_topn_select
    c = fn(_p(a), a.shape[0], N, _p(idx), _p(ta))
    return idx[:c].copy(), ta[:c].copy()


def select_window(n_frames: int, m: int, M: int):
    first = ctypes.c_uint32(0); ln = ctypes.c_uint32(0)
    rc = lib().oracle_select_window(n_frames, m, M, ctypes.byref(first), ctypes.byref(ln))
    if rc != OR_OK:
        raise ValueError(f"select_window rc={rc}")
    return first.value, ln.value


# --------------------------------------------------------------------------- retrieve
@dataclass
class Candidates:
    subspace: np.ndarray
    frame: np.ndarray
    bundle: np.ndarray
    qframe: np.ndarray
    acc: np.ndarray
    dist: np.ndarray
    x: np.ndarray
    y: np.ndarray

    def __len__(self):
        return int(self.frame.shape[0])


def retrieve(sub_sizes, feats, coords, frames, N: int, use_select: bool = False) -> Candidates:
    """Alg. 1: top-N per (bundle, frame, subspace), SPEC order.

    feats [sum sizes][K] f32, coords [sum sizes][2] i32, frames [B][M][K] f32.
    """
    sizes = _c(sub_sizes, np.int64)
    F = _c(feats, np.float32); C = _c(coords, np.int32); Q = _c(frames, np.float32)
    if Q.ndim == 2:
        Q = Q[:, None, :]
    B, M, K = Q.shape
    cap = B * M * int(np.minimum(sizes, N).sum())
    outs = [np.zeros(cap, t) for t in (np.uint32, np.uint32, np.uint32, np.uint32,
                                        np.float32, np.float32, np.int32, np.int32)]
    w = lib().oracle_retrieve(len(sizes), _p(sizes), _p(F), _p(C), K, B, M, _p(Q), N,
                              1 if use_select else 0, *[_p(o) for o in outs], cap)
    if w < 0:
        raise ValueError(f"oracle_retrieve rc={w}")
    return Candidates(*[o[:w] for o in outs])


# --------------------------------------------------------------------------- aggregate
@dataclass
class Estimate:
    x: int
    y: int
    confidence: float
    low_confidence: bool
    ranked_xy: np.ndarray
    ranked_count: np.ndarray
    ranked_circle: np.ndarray
    x_m: float = 0.0      # tile centre in metres: tile_m * x in binary64 (DESIGN R14)
    y_m: float = 0.0


def aggregate(xy, top_c: int = 10, toler_per: float = 0.2, radius_m: float = 3.0,
              tile_m: float = 0.3) -> Estimate:
    """Algorithm 2 on one bundle's candidate tiles xy [n][2]."""
    a = _c(np.asarray(xy).reshape(-1, 2), np.int32)
    n = a.shape[0]
    ox = ctypes.c_int32(0); oy = ctypes.c_int32(0); conf = ctypes.c_double(0)
    low = ctypes.c_int(0); nr = ctypes.c_int(0)
    rxy = np.zeros((max(top_c, 1), 2), np.int32)
    rc_ = np.zeros(max(top_c, 1), np.uint32); rci = np.zeros(max(top_c, 1), np.uint32)
    rc = lib().oracle_aggregate(n, _p(a), top_c, toler_per, radius_m, tile_m,
                                ctypes.byref(ox), ctypes.byref(oy), ctypes.byref(conf),
                                ctypes.byref(low), ctypes.byref(nr), _p(rxy), _p(rc_), _p(rci))
    if rc == OR_ERR_EMPTY:
        raise LookupError("empty candidate set")
    if rc != OR_OK:
        raise ValueError(f"oracle_aggregate rc={rc}")
    k = nr.value
    return Estimate(ox.value, oy.value, conf.value, bool(low.value), rxy[:k].copy(),
                    rc_[:k].copy(), rci[:k].copy(), float(tile_m) * float(ox.value),
                    float(tile_m) * float(oy.value))


def shift_distance(q, d):
    """min over circular shifts s of the fp32 chain sum_w (q[(w+s) mod W] - d[w])^2
    and its smallest argmin (NEXT-1; DESIGN R3/R21)."""
    q = _c(q, np.float32); d = _c(d, np.float32)
    am = ctypes.c_int(0)
    v = lib().oracle_shift_distance(_p(q), _p(d), q.shape[0], ctypes.byref(am))
    return np.float32(v), am.value
