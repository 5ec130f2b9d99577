"""Seeded synthetic input generator "G" -- shared by tests, bench
and smoke.  Holds none of the hot path's arithmetic (no distance, top-N or
aggregation): it only renders poses into descriptors and tiles.  The C/CUDA
source is ``synth.cu``; host rendering uses OpenMP, device rendering a CUDA
kernel (torch supplies the device memory).  Draws are counter-based, so any
slice of a database generates independently of the rest.

Presets C1..C5 follow SURVEY §8(d) (BASELINE.json ``configs``).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "synth.cu")
_LIB = os.path.join(_HERE, "libsynthgen.so")


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call([
            "nvcc", "-O2", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a",
            "-Xcompiler", "-fopenmp,-fPIC", "-shared", "-o", tmp, _SRC, "-lgomp"])
        os.replace(tmp, _LIB)
    return _LIB


class _Spec(ctypes.Structure):
    _fields_ = [("seed", ctypes.c_uint64),
                ("n_floors", ctypes.c_int32), ("paths", ctypes.c_int32),
                ("frames_per_path", ctypes.c_int32),
                ("W", ctypes.c_int32), ("K", ctypes.c_int32), ("n_lm", ctypes.c_int32),
                ("dup_frac", ctypes.c_double), ("floor_reuse", ctypes.c_double),
                ("noise_sigma", ctypes.c_double),
                ("floor_w", ctypes.c_double), ("floor_h", ctypes.c_double),
                ("path_y0", ctypes.c_double), ("path_dy", ctypes.c_double),
                ("atlas_cols", ctypes.c_int32), ("atlas_dx", ctypes.c_int32),
                ("atlas_dy", ctypes.c_int32), ("_pad", ctypes.c_int32)]


class _Point(ctypes.Structure):
    _fields_ = [("floor", ctypes.c_int32), ("x", ctypes.c_double), ("y", ctypes.c_double),
                ("heading", ctypes.c_double), ("noise_key", ctypes.c_uint64)]


POINT_DTYPE = np.dtype([("floor", np.int32), ("x", np.float64), ("y", np.float64),
                        ("heading", np.float64), ("noise_key", np.uint64)], align=True)
assert POINT_DTYPE.itemsize == ctypes.sizeof(_Point)

_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        P, i64, i32, u64, dbl = (ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                                 ctypes.c_uint64, ctypes.c_double)
        SP = ctypes.POINTER(_Spec)
        L.syn_num_entries.argtypes = [SP]; L.syn_num_entries.restype = i64
        L.syn_grid.argtypes = [SP, P, P]; L.syn_grid.restype = None
        L.syn_entry_points.argtypes = [SP, i64, i64, P]; L.syn_entry_points.restype = None
        L.syn_query_points.argtypes = [SP, u64, i32, i64, i32, i32, dbl, P]
        L.syn_query_points.restype = None
        L.syn_render_host.argtypes = [SP, i64, P, P, P, P, P]; L.syn_render_host.restype = None
        L.syn_db_host.argtypes = [SP, i64, i64, P, P]; L.syn_db_host.restype = None
        L.syn_render_device.argtypes = [SP, i64, i32, i64, P, P, P, P]
        L.syn_render_device.restype = i32
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


@dataclass(frozen=True)
class Spec:
    seed: int = 1
    n_floors: int = 1
    paths: int = 5
    frames_per_path: int = 4000
    W: int = 256
    K: int = 64
    n_lm: int = 60
    dup_frac: float = 0.2
    floor_reuse: float = 0.2
    noise_sigma: float = 0.02
    floor_w: float = 200.0
    floor_h: float = 100.0
    path_y0: float = 20.0
    path_dy: float = 15.0
    atlas_cols: int = 64
    atlas_dx: int = 240
    atlas_dy: int = 140

    def c(self) -> _Spec:
        return _Spec(self.seed, self.n_floors, self.paths, self.frames_per_path, self.W,
                     self.K, self.n_lm, self.dup_frac, self.floor_reuse, self.noise_sigma,
                     self.floor_w, self.floor_h, self.path_y0, self.path_dy,
                     self.atlas_cols, self.atlas_dx, self.atlas_dy, 0)

    @property
    def n_entries(self) -> int:
        return self.n_floors * self.paths * self.frames_per_path

    def grid(self):
        gw = ctypes.c_int32(0); gh = ctypes.c_int32(0)
        s = self.c()
        lib().syn_grid(ctypes.byref(s), ctypes.byref(gw), ctypes.byref(gh))
        return gw.value, gh.value


@dataclass(frozen=True)
class Config:
    """One BASELINE.json config."""
    name: str
    spec: Spec
    subspace_sizes: tuple
    n_queries: int           # query frames (M=1) or bundles (M>1)
    M: int = 1
    N: int = 15
    aggregate: bool = True
    query_mode: str = "random"   # "random" positions, or one test "path" video
    note: str = ""


CONFIGS = {
    "C1": Config("C1", Spec(seed=1, n_floors=1, paths=1, frames_per_path=2000, path_y0=50.0),
                 (2000,), n_queries=1, M=1, N=5, query_mode="random",
                 note="tiny: 2,000 features on one corridor path, one query frame, top-5"),
    "C2": Config("C2", Spec(seed=2, n_floors=1, paths=5, frames_per_path=4000),
                 (4000,) * 5, n_queries=1000, M=5, N=15, query_mode="path",
                 note="paper-scale: 20k features, 5 path subspaces, 1,000 bundles of M=5"),
    "C3": Config("C3", Spec(seed=3, n_floors=50, paths=5, frames_per_path=4000),
                 (1_000_000,), n_queries=1024, M=1, N=15,
                 note="1M campus DB, 1,024 query frames"),
    "C4": Config("C4", Spec(seed=4, n_floors=5000, paths=5, frames_per_path=4000),
                 (100_000_000,), n_queries=1024, M=1, N=15,
                 note="100M city DB, 1,024 query frames, sharded over ranks"),
    "C5": Config("C5", Spec(seed=5, n_floors=500, paths=5, frames_per_path=4000),
                 (10_000_000,), n_queries=8, M=1, N=15,
                 note="10M DB, streaming micro-batches of <= 8 frames"),
}


# ------------------------------------------------------------------ host side
def entry_points(spec: Spec, e_begin: int, n: int) -> np.ndarray:
    out = np.zeros(n, POINT_DTYPE)
    s = spec.c()
    lib().syn_entry_points(ctypes.byref(s), e_begin, n, _p(out))
    return out


def query_points(spec: Spec, qseed: int, n: int, mode: str = "random", floor: int = 0,
                 path: int = 0, offset: float = 1.5) -> np.ndarray:
    out = np.zeros(n, POINT_DTYPE)
    s = spec.c()
    lib().syn_query_points(ctypes.byref(s), qseed, 0 if mode == "random" else 1, n, floor,
                           path, offset, _p(out))
    return out


def render_host(spec: Spec, pts: np.ndarray, profiles: bool = False, f64: bool = False):
    """-> dict(desc f32 [n][K], tiles i32 [n][2], profile f64 [n][W]?, desc64?)."""
    n = pts.shape[0]
    pts = np.ascontiguousarray(pts)
    desc = np.zeros((n, spec.K), np.float32)
    tiles = np.zeros((n, 2), np.int32)
    prof = np.zeros((n, spec.W), np.float64) if profiles else None
    d64 = np.zeros((n, spec.K), np.float64) if f64 else None
    s = spec.c()
    lib().syn_render_host(ctypes.byref(s), n, _p(pts), _p(prof) if prof is not None else None,
                          _p(desc), _p(d64) if d64 is not None else None, _p(tiles))
    out = {"desc": desc, "tiles": tiles}
    if prof is not None:
        out["profile"] = prof
    if d64 is not None:
        out["desc64"] = d64
    return out


def db_host(spec: Spec, e_begin: int = 0, n: int | None = None):
    n = spec.n_entries - e_begin if n is None else n
    desc = np.zeros((n, spec.K), np.float32)
    tiles = np.zeros((n, 2), np.int32)
    s = spec.c()
    lib().syn_db_host(ctypes.byref(s), e_begin, n, _p(desc), _p(tiles))
    return desc, tiles


# ------------------------------------------------------------------ device side
def db_device(spec: Spec, e_begin: int, n: int, device, chunk: int = 1 << 22):
    """Render DB entries [e_begin, e_begin+n) straight into device memory."""
    import torch
    desc = torch.empty((n, spec.K), dtype=torch.float32, device=device)
    tiles = torch.empty((n, 2), dtype=torch.int32, device=device)
    s = spec.c()
    stream = torch.cuda.current_stream(device).cuda_stream
    for b in range(0, n, chunk):
        c = min(chunk, n - b)
        rc = lib().syn_render_device(ctypes.byref(s), c, 0, e_begin + b, None,
                                     ctypes.c_void_p(desc[b].data_ptr()),
                                     ctypes.c_void_p(tiles[b].data_ptr()),
                                     ctypes.c_void_p(stream))
        if rc != 0:
            raise RuntimeError(f"syn_render_device failed: {rc}")
    return desc, tiles


def render_device(spec: Spec, pts: np.ndarray, device):
    import torch
    n = pts.shape[0]
    pts_t = torch.from_numpy(np.ascontiguousarray(pts).view(np.uint8)).to(device)
    desc = torch.empty((n, spec.K), dtype=torch.float32, device=device)
    tiles = torch.empty((n, 2), dtype=torch.int32, device=device)
    s = spec.c()
    stream = torch.cuda.current_stream(device).cuda_stream
    rc = lib().syn_render_device(ctypes.byref(s), n, 1, 0, ctypes.c_void_p(pts_t.data_ptr()),
                                 ctypes.c_void_p(desc.data_ptr()),
                                 ctypes.c_void_p(tiles.data_ptr()), ctypes.c_void_p(stream))
    if rc != 0:
        raise RuntimeError(f"syn_render_device failed: {rc}")
    return desc, tiles


# ------------------------------------------------------------------ adversarial
def gflat(n: int, K: int = 64, seed: int = 0, dup_frac: float = 0.01) -> np.ndarray:
    """"Gflat": |N(0,1)|^K rows, L2-normalised, plus exact duplicates
    -- flat spectra that defeat prefix pruning, and ties."""
    rng = np.random.default_rng(seed)
    a = np.abs(rng.standard_normal((n, K)))
    a /= np.linalg.norm(a, axis=1, keepdims=True)
    a = a.astype(np.float32)
    nd = int(n * dup_frac)
    if nd:
        src = rng.integers(0, n, nd); dst = rng.integers(0, n, nd)
        a[dst] = a[src]
    return a


def gather_windows(video: np.ndarray, firsts, length: int) -> np.ndarray:
    """Stack video[first:first+length] for each window start -> [B][length][K].
    Pure indexing; the window rule is computed by the caller with
    the product's ``select_window`` or the oracle's."""
    return np.stack([video[f:f + length] for f in firsts])
