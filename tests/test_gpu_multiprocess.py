"""The sharded path across real processes (the three levels of parallelism,
P:137; candidates collected per query, merged by selectTopCandidates):
two processes, each one rank with its own context and database shard, exchange their
per-rank top-N through a torch.distributed group and end with the global answer --
compared element by element with the oracle run over the WHOLE database (Alg. 1 + Alg. 2),
not with a one-GPU run.

Both ranks share the one GPU a gpurun call provides.  That is safe only because nothing
here makes one rank's kernels wait for the other's: the exchange is gloo (host-staged
copies), so each process's kernels run to completion on their own.  The peer-memory
kernel (ranks spin on each other's flags) and NCCL (refuses two ranks on one device) are
NOT run this way (B200_PROFILING.md: such ranks on one GPU raised Xid 109); they run as
one-process emulations in test_gpu_parity.py / at world 1 in test_gpu_nccl.py."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, out_q):
    import torch.distributed as dist

    import oracle
    import synthgen
    import paper_2006_08861_b200 as ol
    from gpu_helpers import assert_candidates_equal, assert_estimates_equal
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=world)
        cfg = synthgen.CONFIGS["C2"]
        F, C = synthgen.db_host(cfg.spec)
        sizes = cfg.subspace_sizes
        off = np.concatenate([[0], np.cumsum(sizes)])
        rows = np.concatenate([np.arange(off[i] + b, off[i] + b + c) for i, n in enumerate(sizes)
                               for b, c in [ol.shard_range(n, rank, world)]])
        video = synthgen.render_host(cfg.spec, synthgen.query_points(cfg.spec, 31, 200, "path", 0, 1))["desc"]
        eng = ol.Engine(0, coarse_k=16, process_group=dist.group.WORLD, exchange="torch")
        eng.upload(F[rows], C[rows], sizes, cfg.spec.grid())
        checked = 0
        # bundles of M = 5 on the CUDA-core scan, then 64 single frames on the tensor-core filter
        firsts = [ol.select_window(len(video), m, 5)[0] for m in range(0, 200, 3)]
        for Q, tc in ((synthgen.gather_windows(video, firsts, 5), 0), (video[:64][:, None, :], 1)):
            eng.set_option("tc", tc)
            eng.query(torch.from_numpy(np.ascontiguousarray(Q)).cuda(), N=15, aggregate=True)
            got, est = eng.topk(), eng.estimates()
            assert eng.stat("used_tc") == tc
            ref = oracle.retrieve(sizes, F, C, np.ascontiguousarray(Q), 15)
            assert_candidates_equal(got, ref, f"rank {rank} tc={tc}")
            assert_estimates_equal(est, ref, ctx=f"rank {rank} tc={tc}")
            checked += len(got)
        # NEXT-1 across ranks: each rank scores only its own rows, the keys are MIN-combined
        spec = synthgen.Spec(seed=44, n_floors=1, paths=1, frames_per_path=600)
        F1, C1 = synthgen.db_host(spec)
        r = synthgen.render_host(spec, synthgen.query_points(spec, 0, 600, "path", 0, 0), profiles=True)
        P1 = r["profile"].astype(np.float32)
        rq = synthgen.render_host(spec, synthgen.query_points(spec, 5, 4), profiles=True)
        b, c = ol.shard_range(600, rank, world)
        e1 = ol.Engine(0, process_group=dist.group.WORLD, exchange="torch")
        e1.upload(F1[b:b + c], C1[b:b + c], [600], spec.grid())
        e1.upload_profiles(np.ascontiguousarray(P1[b:b + c]))
        e1.query(rq["desc"][:, None, :], N=6, aggregate=False)
        sh, d2 = e1.shift_rescore(rq["profile"].astype(np.float32))
        cands = e1.topk()
        for i in range(len(cands)):
            rd2, rs = oracle.shift_distance(rq["profile"][cands["bundle"][i]].astype(np.float32),
                                            P1[cands["frame"][i]])
            assert (int(sh[i]), d2[i].view(np.uint32)) == (rs, np.float32(rd2).view(np.uint32)), i
        dist.barrier()
        out_q.put((rank, "ok", checked))
    except BaseException as e:   # report, never hang the parent
        import traceback
        out_q.put((rank, "fail", traceback.format_exc()[-3000:]))
    finally:
        try:
            import torch.distributed as dist
            dist.destroy_process_group()
        except Exception:
            pass


def test_two_processes_gloo_exchange_match_oracle():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    try:
        for _ in range(world):
            rank, status, info = q.get(timeout=600)
            res[rank] = (status, info)
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    for rank in range(world):
        status, info = res[rank]
        assert status == "ok", f"rank {rank}:\n{info}"
        assert info > 0
