"""World-size-2 (and 3) CPU tests of the sharded path's host plumbing over gloo:
the product's shard ranges (ol_shard_range) and payload all-gather
(exchange_payloads) with the 16-byte record layout the library emits.  Per-rank
top-N payloads come from the oracle on each shard; merging the gathered
payloads must reproduce the single-process oracle exactly."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import paper_2006_08861_b200 as ol

PAD = 0xFFFFFFFF


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _data():
    rng = np.random.default_rng(5)
    sizes = [1000, 37, 400]
    F = np.abs(rng.standard_normal((sum(sizes), 64))).astype(np.float32)
    F /= np.linalg.norm(F, axis=1, keepdims=True)
    F[10] = F[900]            # duplicates across the shard boundary
    F[999] = F[900]
    C = rng.integers(0, 100, (sum(sizes), 2)).astype(np.int32)
    Q = F[[3, 900, 1020, 1300, 7, 512]].copy()
    Q[0] += 1e-3
    return sizes, F, C, Q.reshape(6, 1, 64)


def _payload(rank, world, sizes, F, C, Q, N):
    """This rank's [frames][n_sub][N] records {acc_bits, frame, x, y} (oracle on its shard)."""
    off = np.concatenate([[0], np.cumsum(sizes)])
    nq = Q.shape[0] * Q.shape[1]
    rec = np.zeros((nq, len(sizes), N, 4), np.uint32)
    rec[..., 0] = PAD
    rec[..., 1] = PAD
    for i, n in enumerate(sizes):
        b, c = ol.shard_range(n, rank, world)
        if c == 0:
            continue
        part = oracle.retrieve([c], F[off[i] + b: off[i] + b + c], C[off[i] + b: off[i] + b + c], Q, N)
        k = 0
        for q in range(nq):
            m = int(min(N, c))
            rec[q, i, :m, 0] = part.acc[k:k + m].view(np.uint32)
            rec[q, i, :m, 1] = part.frame[k:k + m] + b          # global frame index
            rec[q, i, :m, 2] = part.x[k:k + m].view(np.uint32)
            rec[q, i, :m, 3] = part.y[k:k + m].view(np.uint32)
            k += m
    return rec


def _merge(gathered, world, N):
    """N smallest (acc_bits, frame) of the W lists per (frame, subspace)."""
    g = gathered.reshape(world, -1, N, 4)
    out = []
    for j in range(g.shape[1]):
        recs = [tuple(r) for w in range(world) for r in g[w, j] if r[0] != PAD or r[1] != PAD]
        recs.sort(key=lambda r: (int(r[0]), int(r[1])))
        out.append(recs[:N])
    return out


def _worker(rank, world, port, N, result):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    sizes, F, C, Q = _data()
    rec = _payload(rank, world, sizes, F, C, Q, N)
    src = torch.from_numpy(rec.reshape(-1).view(np.uint8).copy())
    assert src.numel() == Q.shape[0] * len(sizes) * N * ol.PAYLOAD_RECORD_BYTES
    dst = torch.empty(src.numel() * world, dtype=torch.uint8)
    ol.exchange_payloads(src, dst)
    merged = _merge(dst.numpy().view(np.uint32), world, N)
    result[rank] = merged
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_sharded_merge_equals_single(world):
    N = 15
    port = _free_port()
    mgr = mp.Manager()
    result = mgr.dict()
    mp.spawn(_worker, args=(world, port, N, result), nprocs=world, join=True)
    sizes, F, C, Q = _data()
    ref = oracle.retrieve(sizes, F, C, Q, N)
    # expected per (frame, subspace) lists from the single-process oracle
    exp = []
    k = 0
    for q in range(Q.shape[0]):
        for i, n in enumerate(sizes):
            m = min(N, n)
            exp.append([(int(a), int(f), int(x) & 0xFFFFFFFF, int(y) & 0xFFFFFFFF)
                        for a, f, x, y in zip(ref.acc[k:k + m].view(np.uint32), ref.frame[k:k + m],
                                              ref.x[k:k + m], ref.y[k:k + m])])
            k += m
    for r in range(world):
        got = [[tuple(int(v) for v in t) for t in lst] for lst in result[r]]
        assert got == exp, f"rank {r}"


def _handle_worker(rank, world, port, result):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    h = bytes([rank]) * 32 + bytes(range(32))          # a 64-byte stand-in for a CUDA IPC handle
    result[rank] = ol.gather_handles(h)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_p2p_handle_exchange(world):
    """The peer-memory exchange's setup (Engine exchange="p2p"): every rank receives all
    ranks' 64-byte mailbox handles in rank order, as ol_p2p_connect expects."""
    port = _free_port()
    mgr = mp.Manager()
    result = mgr.dict()
    mp.spawn(_handle_worker, args=(world, port, result), nprocs=world, join=True)
    want = b"".join(bytes([r]) * 32 + bytes(range(32)) for r in range(world))
    for r in range(world):
        assert result[r] == want
