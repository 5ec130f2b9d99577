"""omniloc -- B200-native hot path of arXiv 2006.08861 (Hu, Zhu, Zhang, ICMR'16).

Thin Python binding over the C-ABI in ``include/omniloc.h`` (``libomniloc.so``):
argument marshalling only.  Every step of the path -- distance chain, coarse
pruning, fine completion, top-N selection, merges and Algorithm 2 -- runs in the
library's sm_100a kernels.  PyTorch provides device memory, the CUDA stream and
(for sharded databases) the ``torch.distributed`` all-gather of the per-rank
top-N payloads (only in the "torch" exchange mode; the default "nccl" mode runs the
collectives inside the library on its own communicator, torch only broadcasts the
NCCL unique id).  There is no CPU fallback: if the library or a GPU is missing,
``Engine`` raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

__all__ = ["Engine", "OmnilocError", "lib", "select_window", "shard_range", "CANDIDATE_DTYPE",
           "ESTIMATE_DTYPE", "PAYLOAD_RECORD_BYTES", "build"]

_HERE = os.path.dirname(os.path.abspath(__file__))
# OL_LIB=checked loads the bounds-checked build (tests / tools/sanitize_cases.py only)
# (OL_LIB_PATH: another build of the same library, for A/B timing tools)
LIB_PATH = os.environ.get("OL_LIB_PATH") or os.path.join(
    _HERE, "libomniloc_checked.so" if os.environ.get("OL_LIB") == "checked" else "libomniloc.so")

OL_OK, OL_ERR_INVALID_ARGUMENT, OL_ERR_DIMENSION_MISMATCH, OL_ERR_NONFINITE = 0, -1, -2, -3
OL_ERR_OUT_OF_RANGE, OL_ERR_OOM, OL_ERR_CUDA, OL_ERR_NOT_READY, OL_ERR_EMPTY = -4, -5, -6, -7, -8
OL_ERR_NCCL = -9
NCCL_ID_BYTES = 128
K = 64
MAX_TOP_C = 64
PAYLOAD_RECORD_BYTES = 16

_NAMES = {0: "OK", -1: "INVALID_ARGUMENT", -2: "DIMENSION_MISMATCH", -3: "NONFINITE",
          -4: "OUT_OF_RANGE", -5: "OOM", -6: "CUDA", -7: "NOT_READY", -8: "EMPTY", -9: "NCCL"}


class OmnilocError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"OL_ERR_{_NAMES.get(status, status)}: {msg}")
        self.status = status


class ol_config(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int32), ("rank", ctypes.c_int32), ("world", ctypes.c_int32),
                ("cuda_stream", ctypes.c_void_p), ("K", ctypes.c_uint32), ("coarse_k", ctypes.c_uint32),
                ("nccl_unique_id", ctypes.c_void_p)]


class ol_db_desc(ctypes.Structure):
    _fields_ = [("n_subspaces", ctypes.c_uint32), ("global_sizes", ctypes.c_void_p),
                ("shard_begin", ctypes.c_void_p), ("shard_count", ctypes.c_void_p),
                ("features", ctypes.c_void_p), ("coords", ctypes.c_void_p),
                ("grid_w", ctypes.c_int32), ("grid_h", ctypes.c_int32), ("on_device", ctypes.c_int32)]


class ol_params(ctypes.Structure):
    _fields_ = [("N", ctypes.c_uint32), ("top_c", ctypes.c_uint32), ("toler_per", ctypes.c_double),
                ("radius_m", ctypes.c_double), ("tile_m", ctypes.c_double)]


CANDIDATE_DTYPE = np.dtype([("subspace", np.uint32), ("frame", np.uint32), ("bundle", np.uint32),
                            ("query_frame", np.uint32), ("dist2", np.float32), ("dist", np.float32),
                            ("x", np.int32), ("y", np.int32)])
RANKED_DTYPE = np.dtype([("x", np.int32), ("y", np.int32), ("count", np.uint32), ("circle", np.uint32)])
ESTIMATE_DTYPE = np.dtype([("x", np.int32), ("y", np.int32), ("x_m", np.float64), ("y_m", np.float64),
                           ("confidence", np.float64), ("low_confidence", np.uint32),
                           ("n_ranked", np.uint32), ("total", np.uint32), ("_pad", np.uint32),
                           ("ranked", RANKED_DTYPE, (MAX_TOP_C,))])
assert CANDIDATE_DTYPE.itemsize == 32 and ESTIMATE_DTYPE.itemsize == 48 + 16 * MAX_TOP_C

_lib = None


def build(force: bool = False) -> str:
    from . import _build
    return _build.build(force=force)


def lib():
    """Load libomniloc.so (raises if it was never built -- no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run paper_2006_08861_b200.build() "
                              "(or __graft_entry__.build()) first; there is no CPU fallback")
        # torch first: its NCCL (libnccl.so.2) is then the one already in the process, and the
        # library's on-demand dlopen of NCCL resolves to it rather than to another copy
        import torch  # noqa: F401
        L = ctypes.CDLL(LIB_PATH)
        P, u32, u64, i32, i64 = (ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int32,
                                 ctypes.c_int64)
        sig = {
            "ol_create": ([ctypes.POINTER(ol_config), ctypes.POINTER(P)], i32),
            "ol_destroy": ([P], None),
            "ol_nccl_unique_id": ([P], i32),
            "ol_last_error": ([P], ctypes.c_char_p),
            "ol_set_stream": ([P, P], i32),
            "ol_shard_range": ([u64, i32, i32, ctypes.POINTER(u64), ctypes.POINTER(u64)], i32),
            "ol_upload_db": ([P, ctypes.POINTER(ol_db_desc)], i32),
            "ol_query": ([P, u32, u32, P, i32, ctypes.POINTER(ol_params), i32], i32),
            "ol_payload": ([P, ctypes.POINTER(P), ctypes.POINTER(u64)], i32),
            "ol_thresholds": ([P, ctypes.POINTER(P), ctypes.POINTER(u64)], i32),
            "ol_payload_copy": ([P, P], i32),
            "ol_finalize": ([P, P, i32], i32),
            "ol_p2p_open": ([P, i32, i32, u64, P], i32),
            "ol_p2p_connect": ([P, P], i32),
            "ol_p2p_finalize": ([P], i32),
            "ol_p2p_emulate": ([ctypes.POINTER(P), i32], i32),
            "ol_tau_share_emulate": ([ctypes.POINTER(P), i32], i32),
            "ol_candidate_count": ([P, ctypes.POINTER(u64)], i32),
            "ol_get_topk": ([P, P, u64, ctypes.POINTER(u64)], i32),
            "ol_topk_device": ([P, ctypes.POINTER(P), ctypes.POINTER(u64)], i32),
            "ol_get_estimates": ([P, P, u32], i32),
            "ol_get_results": ([P, P, u64, ctypes.POINTER(u64), P, u32], i32),
            "ol_aggregate": ([P, u32, P, P, i32, ctypes.POINTER(ol_params), P], i32),
            "ol_select_window": ([u32, u32, u32, ctypes.POINTER(u32), ctypes.POINTER(u32)], i32),
            "ol_set_option": ([P, ctypes.c_char_p, i64], i32),
            "ol_upload_profiles": ([P, P, u32, i32], i32),
            "ol_shift_rescore": ([P, P, i32], i32),
            "ol_shift_rescore_cands": ([P, P, P, u32, i32], i32),
            "ol_shift_keys": ([P, ctypes.POINTER(P), ctypes.POINTER(u64)], i32),
            "ol_get_shifts": ([P, P, P, u64], i32),
            "ol_shift_keys_copy": ([P, P], i32),
            "ol_get_stat": ([P, ctypes.c_char_p, ctypes.POINTER(i64)], i32),
            "ol_extract_features": ([P, P, u64, u32, i32, P, P, P, P], i32),
        }
        for name, (args, res) in sig.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


def _check(status: int, ctx=None):
    if status != OL_OK:
        raise OmnilocError(status, lib().ol_last_error(ctx).decode())


def select_window(n_frames: int, m: int, M: int):
    """selectNearbyFrames (Alg. 1): -> (first, length)."""
    f = ctypes.c_uint32(); n = ctypes.c_uint32()
    _check(lib().ol_select_window(n_frames, m, M, ctypes.byref(f), ctypes.byref(n)))
    return f.value, n.value


def shard_range(n: int, rank: int, world: int):
    b = ctypes.c_uint64(); c = ctypes.c_uint64()
    _check(lib().ol_shard_range(n, rank, world, ctypes.byref(b), ctypes.byref(c)))
    return b.value, c.value


def _ptr(x):
    """(pointer, on_device) of a contiguous torch tensor or numpy array."""
    if isinstance(x, np.ndarray):
        assert x.flags["C_CONTIGUOUS"]
        return x.ctypes.data, 0
    assert x.is_contiguous()
    return x.data_ptr(), int(x.is_cuda)


@dataclass
class Params:
    N: int = 15
    top_c: int = 10
    toler_per: float = 0.2
    radius_m: float = 3.0
    tile_m: float = 0.3

    def c(self) -> ol_params:
        return ol_params(self.N, self.top_c, self.toler_per, self.radius_m, self.tile_m)


class Engine:
    """One context on one GPU: upload a (sharded) feature database, query bundles.

    ``process_group``: a torch.distributed group whose ranks each hold one shard.
    ``exchange`` picks how the ranks' top-N meet:

    - ``"nccl"`` (default): the library owns a NCCL communicator (rank 0's
      ``ol_nccl_unique_id`` broadcast over the group, the only thing torch does) and
      ``ol_query`` runs the threshold MIN all-reduce, the all-gather and the merge
      itself.  ``comm=True`` also builds it at world 1 (a 1-rank communicator).
    - ``"torch"``: ``ol_query`` returns this rank's payload; the binding all-gathers it
      with ``torch.distributed`` (any backend: gloo stages through the host) and calls
      ``ol_finalize``.
    - ``"p2p"``: one kernel exchanges and merges over NVLink peer memory (mailbox
      handles are exchanged through the group once).
    """

    def __init__(self, device: int = 0, coarse_k: int = 16, process_group=None, rank: int | None = None,
                 world: int | None = None, stream=None, exchange: str = "nccl", comm: bool | None = None):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("omniloc needs a CUDA device (no CPU fallback)")
        self._torch = torch
        self.device = torch.device("cuda", device)
        self.group = process_group
        if process_group is not None:
            import torch.distributed as dist
            rank = dist.get_rank(process_group)
            world = dist.get_world_size(process_group)
        self.rank = 0 if rank is None else rank
        self.world = 1 if world is None else world
        self._stream = stream
        if exchange not in ("nccl", "torch", "p2p"):
            raise ValueError("exchange must be 'nccl', 'torch' or 'p2p'")
        self.exchange = exchange
        if comm is None:
            comm = exchange == "nccl" and self.world > 1
        if comm and exchange != "nccl":
            raise ValueError("comm=True needs exchange='nccl'")
        if self.world > 1 and exchange == "nccl" and not comm:
            raise ValueError("exchange='nccl' at world > 1 needs the library communicator")
        L = lib()
        uid = None
        if comm:
            uid = ctypes.create_string_buffer(NCCL_ID_BYTES)
            if self.rank == 0:
                _check(L.ol_nccl_unique_id(uid))
            if self.world > 1:
                if process_group is None:
                    raise ValueError("a NCCL communicator over world > 1 needs a process group")
                import torch.distributed as dist
                obj = [uid.raw if self.rank == 0 else None]
                dist.broadcast_object_list(obj, src=dist.get_global_rank(process_group, 0), group=process_group)
                uid = ctypes.create_string_buffer(obj[0], NCCL_ID_BYTES)
        self.comm = bool(comm)
        torch.cuda.set_device(self.device)
        cfg = ol_config(device, self.rank, self.world, self._stream_ptr(), K, coarse_k,
                        ctypes.cast(uid, ctypes.c_void_p) if uid is not None else None)
        h = ctypes.c_void_p()
        _check(L.ol_create(ctypes.byref(cfg), ctypes.byref(h)))
        self._h = h
        self.params = Params()
        self._gather_buf = None
        self._payload_buf = None
        self._mbox_bytes = 0

    def _stream_ptr(self):
        if self._stream is not None:
            return self._stream.cuda_stream
        return self._torch.cuda.current_stream(self.device).cuda_stream

    def close(self):
        if getattr(self, "_h", None):
            lib().ol_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _ck(self, status):
        if status != OL_OK:
            raise OmnilocError(status, lib().ol_last_error(self._h).decode())

    def sync_stream(self):
        """Order the library's work on torch's current stream (or the given one)."""
        s = self._stream_ptr()
        if s != getattr(self, "_bound_stream", None):
            self._ck(lib().ol_set_stream(self._h, ctypes.c_void_p(s)))
            self._bound_stream = s

    # ---------------------------------------------------------------- database
    def upload(self, features, coords, subspace_sizes, grid, shard_begin=None, shard_count=None):
        """features [rows][64] f32, coords [rows][2] i32 (this rank's rows, subspace order);
        subspace_sizes: global |n_i|; grid: (grid_w, grid_h)."""
        self.sync_stream()
        sizes = np.ascontiguousarray(subspace_sizes, np.uint64)
        fp, fdev = _ptr(features)
        cp, cdev = _ptr(coords)
        if fdev != cdev:
            raise ValueError("features and coords must both be host or both device")
        sb = sc = None
        if shard_begin is not None:
            sb = np.ascontiguousarray(shard_begin, np.uint64)
            sc = np.ascontiguousarray(shard_count, np.uint64)
        desc = ol_db_desc(len(sizes), sizes.ctypes.data, sb.ctypes.data if sb is not None else None,
                          sc.ctypes.data if sc is not None else None, fp, cp, int(grid[0]), int(grid[1]),
                          fdev)
        self._ck(lib().ol_upload_db(self._h, ctypes.byref(desc)))
        self.sizes = sizes

    # ---------------------------------------------------------------- query
    def query(self, frames, N: int | None = None, aggregate: bool = True, params: Params | None = None,
              M: int | None = None, exchange: bool = True):
        """frames [B][M][64] (or [B][64] for M=1) f32, host (numpy / pinned torch) or device.
        Runs Alg. 1 + Alg. 2; results via topk() / estimates().  With world > 1 and
        ``exchange`` the per-rank payloads are all-gathered over the process group
        and merged; with ``exchange=False`` the caller gathers (payload() /
        finalize_gathered())."""
        p = params or self.params
        if N is not None:
            p = Params(N, p.top_c, p.toler_per, p.radius_m, p.tile_m)
        shape = tuple(frames.shape)
        if len(shape) == 2:
            B, Mq = shape[0], 1
        else:
            B, Mq = shape[0], shape[1]
        if M is not None:
            Mq = M
        self.sync_stream()
        fp, fdev = _ptr(frames)
        pc = p.c()
        self._ck(lib().ol_query(self._h, B, Mq, ctypes.c_void_p(fp), fdev, ctypes.byref(pc),
                                1 if aggregate else 0))
        if self.world > 1 and exchange and not self.comm:   # (with a communicator: done in ol_query)
            if self.exchange == "p2p":
                self._p2p_finalize()
            else:
                self._exchange_and_finalize()
        self._last = (B, Mq, p, aggregate)

    # ---------------------------------------------------------------- peer-memory exchange
    def p2p_open(self, world: int, rank: int, max_payload_bytes: int) -> bytes:
        """Allocate this rank's mailbox; returns its 64-byte CUDA IPC handle."""
        h = ctypes.create_string_buffer(64)
        self._ck(lib().ol_p2p_open(self._h, world, rank, max_payload_bytes, h))
        self._mbox_bytes = max_payload_bytes
        return h.raw

    def p2p_connect(self, handles: bytes):
        """Open the peers' mailboxes (world x 64 bytes, rank order)."""
        buf = ctypes.create_string_buffer(handles, len(handles))
        self._ck(lib().ol_p2p_connect(self._h, buf))

    def _p2p_finalize(self):
        """Cross-GPU merge over peer memory (one kernel: push to every rank's mailbox,
        signal, wait, merge).  The first call, and a payload larger than the mailbox,
        (re)build the mailboxes collectively: every rank has the same payload size."""
        ptr = ctypes.c_void_p(); nbytes = ctypes.c_uint64()
        self._ck(lib().ol_payload(self._h, ctypes.byref(ptr), ctypes.byref(nbytes)))
        if nbytes.value > self._mbox_bytes:
            cap = max(nbytes.value, 2 * self._mbox_bytes)
            cap = (cap + 15) // 16 * 16
            handle = self.p2p_open(self.world, self.rank, cap)
            self.p2p_connect(gather_handles(handle, self.group))
        self._ck(lib().ol_p2p_finalize(self._h))

    def _exchange_and_finalize(self):
        """Cross-GPU merge: all-gather the per-rank top-N payloads
        through torch.distributed (NCCL over NVLink on GPUs), merge in-library."""
        torch = self._torch
        ptr = ctypes.c_void_p(); nbytes = ctypes.c_uint64()
        self._ck(lib().ol_payload(self._h, ctypes.byref(ptr), ctypes.byref(nbytes)))
        n = nbytes.value
        if self._payload_buf is None or self._payload_buf.numel() < n:
            self._payload_buf = torch.empty(n, dtype=torch.uint8, device=self.device)
            self._gather_buf = torch.empty(n * self.world, dtype=torch.uint8, device=self.device)
        src = self._payload_buf[:n]
        dst = self._gather_buf[: n * self.world]
        self._ck(lib().ol_payload_copy(self._h, ctypes.c_void_p(src.data_ptr())))
        exchange_payloads(src, dst, self.group)
        self._ck(lib().ol_finalize(self._h, ctypes.c_void_p(dst.data_ptr()), self.world))

    def finalize_gathered(self, gathered):
        """Finalize with payloads gathered by the caller (device tensor, rank order)."""
        self._ck(lib().ol_finalize(self._h, ctypes.c_void_p(gathered.data_ptr()), self.world))

    def thresholds(self):
        """Zero-copy device view (torch int32, [frames * subspaces]) of the last query's
        pruning thresholds (acc bits of non-negative floats, < 2^31, as int32); see ol_thresholds."""
        ptr = ctypes.c_void_p(); n = ctypes.c_uint64()
        self._ck(lib().ol_thresholds(self._h, ctypes.byref(ptr), ctypes.byref(n)))

        class _View:
            __cuda_array_interface__ = {"shape": (n.value,), "typestr": "<i4", "data": (ptr.value, False),
                                        "version": 3, "strides": None}
        return self._torch.as_tensor(_View(), device=self.device)

    def payload(self):
        """This rank's payload as a new device uint8 tensor."""
        ptr = ctypes.c_void_p(); nbytes = ctypes.c_uint64()
        self._ck(lib().ol_payload(self._h, ctypes.byref(ptr), ctypes.byref(nbytes)))
        t = self._torch.empty(nbytes.value, dtype=self._torch.uint8, device=self.device)
        self._ck(lib().ol_payload_copy(self._h, ctypes.c_void_p(t.data_ptr())))
        return t

    # ---------------------------------------------------------------- results
    def candidate_count(self) -> int:
        n = ctypes.c_uint64()
        self._ck(lib().ol_candidate_count(self._h, ctypes.byref(n)))
        return n.value

    def topk(self, out: np.ndarray | None = None) -> np.ndarray:
        n = self.candidate_count()
        if out is None:
            out = np.empty(n, CANDIDATE_DTYPE)
        w = ctypes.c_uint64()
        self._ck(lib().ol_get_topk(self._h, ctypes.c_void_p(out.ctypes.data), out.shape[0], ctypes.byref(w)))
        return out[: w.value]

    def topk_into(self, pinned) -> int:
        """D2H of the candidates into a (pinned) torch uint8 host tensor; returns bytes."""
        n = self.candidate_count()
        w = ctypes.c_uint64()
        self._ck(lib().ol_get_topk(self._h, ctypes.c_void_p(pinned.data_ptr()),
                                   pinned.numel() // CANDIDATE_DTYPE.itemsize, ctypes.byref(w)))
        return n * CANDIDATE_DTYPE.itemsize

    def estimates_into(self, pinned) -> int:
        """D2H of the estimates into a (pinned) torch uint8 host tensor; returns bytes."""
        B = self._last[0]
        self._ck(lib().ol_get_estimates(self._h, ctypes.c_void_p(pinned.data_ptr()),
                                        pinned.numel() // ESTIMATE_DTYPE.itemsize))
        return B * ESTIMATE_DTYPE.itemsize

    def results_into(self, cand_pinned, est_pinned=None) -> tuple:
        """D2H of the candidates and (if given) the estimates into (pinned) torch uint8 host
        tensors with one synchronisation (ol_get_results); returns (candidate, estimate) bytes."""
        w = ctypes.c_uint64()
        est_p = ctypes.c_void_p(est_pinned.data_ptr()) if est_pinned is not None else None
        est_cap = est_pinned.numel() // ESTIMATE_DTYPE.itemsize if est_pinned is not None else 0
        self._ck(lib().ol_get_results(self._h, ctypes.c_void_p(cand_pinned.data_ptr()),
                                      cand_pinned.numel() // CANDIDATE_DTYPE.itemsize, ctypes.byref(w), est_p, est_cap))
        return w.value * CANDIDATE_DTYPE.itemsize, (self._last[0] * ESTIMATE_DTYPE.itemsize if est_pinned is not None else 0)

    def topk_device(self):
        """(device pointer, count) of the candidate array (owned by the engine)."""
        p = ctypes.c_void_p(); n = ctypes.c_uint64()
        self._ck(lib().ol_topk_device(self._h, ctypes.byref(p), ctypes.byref(n)))
        return p.value, n.value

    def estimates(self) -> np.ndarray:
        B = self._last[0]
        out = np.empty(B, ESTIMATE_DTYPE)
        self._ck(lib().ol_get_estimates(self._h, ctypes.c_void_p(out.ctypes.data), B))
        return out

    def aggregate(self, xy, offsets, params: Params | None = None) -> np.ndarray:
        """Algorithm 2 alone: bundle b owns xy[offsets[b]:offsets[b+1]].  xy / offsets are
        host arrays, or both device tensors (int32 [n][2], uint32-valued int32 [nb+1])."""
        p = (params or self.params).c()
        if hasattr(xy, "is_cuda") and xy.is_cuda:
            xy_p, dev = _ptr(xy.contiguous())
            off_p, odev = _ptr(offsets.contiguous())
            assert odev, "offsets must live with xy"
            nb = int(offsets.shape[0]) - 1
        else:
            xy = np.ascontiguousarray(xy, np.int32).reshape(-1, 2)
            off = np.ascontiguousarray(offsets, np.uint32)
            xy_p, off_p, dev, nb = xy.ctypes.data, off.ctypes.data, 0, off.shape[0] - 1
        out = np.empty(nb, ESTIMATE_DTYPE)
        self.sync_stream()
        self._ck(lib().ol_aggregate(self._h, nb, ctypes.c_void_p(off_p), ctypes.c_void_p(xy_p), dev,
                                    ctypes.byref(p), ctypes.c_void_p(out.ctypes.data)))
        return out

    # ---------------------------------------------------------------- NEXT-1
    def upload_profiles(self, profiles):
        """This rank's database profiles [rows][W] fp32 (same order as upload())."""
        self.sync_stream()
        pp, pdev = _ptr(profiles)
        self._ck(lib().ol_upload_profiles(self._h, ctypes.c_void_p(pp), int(profiles.shape[1]), pdev))

    def shift_rescore(self, query_profiles):
        """Heading of every candidate of the last query: -> (shift u32, dist2 f32) arrays.
        query_profiles [B][M][W] (or [B*M][W]) fp32, host or device.  With world > 1 the
        per-rank keys are MIN-reduced over the process group."""
        self.sync_stream()
        qp, qdev = _ptr(query_profiles)
        self._ck(lib().ol_shift_rescore(self._h, ctypes.c_void_p(qp), qdev))
        n = self.candidate_count()
        if self.world > 1 and not self.comm:   # (with a communicator ol_shift_rescore MIN-reduces)
            torch = self._torch
            keys = torch.empty(max(n, 1), dtype=torch.int64, device=self.device)
            self._ck(lib().ol_shift_keys_copy(self._h, ctypes.c_void_p(keys.data_ptr())))
            min_reduce(keys, self.group)
            keys = keys[:n]
            k = keys.cpu().numpy().view(np.uint64)
            shift = (k & 0xFFFFFFFF).astype(np.uint32)
            dist2 = (k >> 32).astype(np.uint32).view(np.float32)
            return shift, dist2
        shift = np.empty(n, np.uint32); dist2 = np.empty(n, np.float32)
        self._ck(lib().ol_get_shifts(self._h, ctypes.c_void_p(shift.ctypes.data),
                                     ctypes.c_void_p(dist2.ctypes.data), n))
        return shift, dist2

    def shift_rescore_cands(self, query_profiles, cand_profiles, fetch: bool = True):
        """Heading of every candidate from caller-supplied candidate profiles [n_cand][W] (candidate
        order) and query profiles [B*M][W], both host or both device fp32 -> (shift, dist2) when
        fetch, else nothing (results stay on the device: ol_shift_keys)."""
        self.sync_stream()
        qp, qdev = _ptr(query_profiles)
        cp, cdev = _ptr(cand_profiles)
        if qdev != cdev:
            raise ValueError("query and candidate profiles must both be host or both device")
        self._ck(lib().ol_shift_rescore_cands(self._h, ctypes.c_void_p(qp), ctypes.c_void_p(cp),
                                              int(cand_profiles.shape[-1]), qdev))
        if not fetch:
            return None
        n = self.candidate_count()
        shift = np.empty(n, np.uint32); dist2 = np.empty(n, np.float32)
        self._ck(lib().ol_get_shifts(self._h, ctypes.c_void_p(shift.ctypes.data),
                                     ctypes.c_void_p(dist2.ctypes.data), n))
        return shift, dist2

    def extract_features(self, profiles, want64: bool = False, want_profiles: bool = False):
        """Descriptors of omnidirectional profiles (NEXT-3): [n][W] binary64,
        host numpy or device torch -> (fp32 [n][64], degenerate bool [n]) plus binary64 [n][64]
        if want64, plus the NEXT-1 stored profiles fp32 [n][W] ((x - mean)/||m||) if
        want_profiles; same residency as the input.  Every step runs in the library's kernels."""
        n, W = int(profiles.shape[0]), int(profiles.shape[1])
        pp, pdev = _ptr(profiles)
        if pdev:
            torch = self._torch
            self.sync_stream()
            o32 = torch.empty((n, 64), dtype=torch.float32, device=profiles.device)
            o64 = torch.empty((n, 64), dtype=torch.float64, device=profiles.device) if want64 else None
            po = torch.empty((n, W), dtype=torch.float32, device=profiles.device) if want_profiles else None
            deg = torch.empty(n, dtype=torch.uint8, device=profiles.device)
            self._ck(lib().ol_extract_features(self._h, ctypes.c_void_p(pp), n, W, 1,
                                               ctypes.c_void_p(o32.data_ptr()),
                                               ctypes.c_void_p(o64.data_ptr() if want64 else None),
                                               ctypes.c_void_p(deg.data_ptr()),
                                               ctypes.c_void_p(po.data_ptr() if want_profiles else None)))
            deg = deg.bool()
        else:
            o32 = np.empty((n, 64), np.float32)
            o64 = np.empty((n, 64), np.float64) if want64 else None
            po = np.empty((n, W), np.float32) if want_profiles else None
            deg = np.empty(n, np.uint8)
            self._ck(lib().ol_extract_features(self._h, ctypes.c_void_p(pp), n, W, 0,
                                               ctypes.c_void_p(o32.ctypes.data),
                                               ctypes.c_void_p(o64.ctypes.data if want64 else None),
                                               ctypes.c_void_p(deg.ctypes.data),
                                               ctypes.c_void_p(po.ctypes.data if want_profiles else None)))
            deg = deg.astype(bool)
        out = (o32, deg)
        if want64:
            out += (o64,)
        if want_profiles:
            out += (po,)
        return out

    def set_option(self, key: str, value: int):
        self._ck(lib().ol_set_option(self._h, key.encode(), int(value)))

    def stat(self, key: str) -> int:
        v = ctypes.c_int64()
        self._ck(lib().ol_get_stat(self._h, key.encode(), ctypes.byref(v)))
        return v.value


def gather_handles(handle: bytes, group=None) -> bytes:
    """All ranks' 64-byte mailbox handles, concatenated in rank order (host objects
    over the process group: gloo or NCCL)."""
    import torch.distributed as dist
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, handle, group=group)
    return b"".join(out)


def p2p_emulate(engines):
    """Tests: the peer-memory exchange kernel emulating len(engines) ranks on one GPU
    as one cooperative launch (engine g = rank g, each after p2p_open(world, g, ..)
    and its own query(..., exchange=False))."""
    arr = (ctypes.c_void_p * len(engines))(*[e._h.value for e in engines])
    _check(lib().ol_p2p_emulate(arr, len(engines)), engines[0]._h)


def _host_staged(t, group) -> bool:
    """gloo moves host tensors only: device tensors are staged through the host."""
    import torch.distributed as dist
    return t.is_cuda and dist.get_backend(group) == "gloo"


def tau_share_emulate(engines):
    """Tests / measurements: link engines on one GPU so their tensor-core scans share
    thresholds as NCCL-mode ranks do over peer memory (ol_tau_share_emulate)."""
    arr = (ctypes.c_void_p * len(engines))(*[e._h.value for e in engines])
    _check(lib().ol_tau_share_emulate(arr, len(engines)), engines[0]._h)


def exchange_payloads(src, dst, group=None):
    """All-gather equal-size uint8 payload tensors in rank order (NCCL on CUDA
    tensors; gloo through host copies).  The "torch" exchange mode's collective (§8e)."""
    import torch.distributed as dist
    if _host_staged(src, group):
        h = dst.new_empty(dst.shape, device="cpu")
        dist.all_gather_into_tensor(h, src.cpu(), group=group)
        dst.copy_(h)
        return dst
    dist.all_gather_into_tensor(dst, src, group=group)
    return dst


def min_reduce(t, group=None):
    """In-place MIN all-reduce (the "torch" mode's combine of NEXT-1 shift keys)."""
    import torch.distributed as dist
    if _host_staged(t, group):
        h = t.cpu()
        dist.all_reduce(h, op=dist.ReduceOp.MIN, group=group)
        t.copy_(h)
        return t
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    return t
