"""The in-library collective ("the collective is internal when world > 1"):
a context created with a NCCL unique id owns its communicator, and ol_query runs the
threshold MIN all-reduce, the all-gather of the per-rank top-N and the merge on the
context stream.  One gpurun call has one GPU and NCCL will not put two ranks on one
device, so this runs the same code path on a 1-rank communicator; results must equal
the oracle's (Alg. 1; Alg. 2) on both scan paths, and NEXT-1's key
all-reduce must leave the oracle's shift distances."""
import ctypes

import numpy as np
import pytest
import torch

import oracle
import synthgen
import paper_2006_08861_b200 as ol
from gpu_helpers import assert_candidates_equal, assert_estimates_equal

pytestmark = pytest.mark.gpu


def test_unique_id_and_version():
    uid = ctypes.create_string_buffer(ol.NCCL_ID_BYTES)
    assert ol.lib().ol_nccl_unique_id(uid) == 0
    assert any(uid.raw)
    e = ol.Engine(0, comm=True)
    assert e.stat("nccl") == 1
    assert e.stat("nccl_version") >= 22700
    assert ol.Engine(0).stat("nccl") == 0


@pytest.mark.parametrize("tc", [0, 1])
def test_nccl_world1_query_matches_oracle(tc):
    cfg = synthgen.CONFIGS["C2"]
    F, C = synthgen.db_host(cfg.spec)
    video = synthgen.render_host(cfg.spec, synthgen.query_points(cfg.spec, 23, 300, "path", 0, 3))["desc"]
    firsts = [ol.select_window(len(video), m, 5)[0] for m in range(0, 300, 7)]
    Q = synthgen.gather_windows(video, firsts, 5)
    e = ol.Engine(0, coarse_k=16, comm=True)
    e.upload(torch.from_numpy(F).cuda(), torch.from_numpy(C).cuda(), cfg.subspace_sizes, cfg.spec.grid())
    e.set_option("tc", tc)
    ref = oracle.retrieve(cfg.subspace_sizes, F, C, Q, 15)
    for it in range(3):   # repeated queries reuse the communicator and the gather buffer
        e.query(torch.from_numpy(Q).cuda(), N=15, aggregate=True)
        assert e.stat("used_tc") == tc
        assert_candidates_equal(e.topk(), ref, f"nccl world 1 tc={tc} it={it}")
        assert_estimates_equal(e.estimates(), ref, ctx=f"nccl world 1 tc={tc}")


def test_nccl_world1_shift_keys_all_reduce():
    spec = synthgen.Spec(seed=45, n_floors=1, paths=1, frames_per_path=500)
    F, C = synthgen.db_host(spec)
    P = synthgen.render_host(spec, synthgen.query_points(spec, 0, 500, "path", 0, 0),
                             profiles=True)["profile"].astype(np.float32)
    r = synthgen.render_host(spec, synthgen.query_points(spec, 6, 5), profiles=True)
    e = ol.Engine(0, comm=True)
    e.upload(F, C, [500], spec.grid())
    e.upload_profiles(P)
    e.query(r["desc"][:, None, :], N=4, aggregate=False)
    sh, d2 = e.shift_rescore(r["profile"].astype(np.float32))
    cands = e.topk()
    for i in range(len(cands)):
        rd2, rs = oracle.shift_distance(r["profile"][cands["bundle"][i]].astype(np.float32), P[cands["frame"][i]])
        assert (int(sh[i]), d2[i].view(np.uint32)) == (rs, np.float32(rd2).view(np.uint32))


def test_plain_c_caller_world1_nccl(tmp_path):
    """A plain C program (tests/c/c_caller.c: no Python, no torch, the system NCCL loaded by the
    library itself) creates a world-1 context with a NCCL id, queries bundles with Alg. 2 and
    gets candidates and estimates equal to the oracle's."""
    import subprocess
    from test_abi import _build_c_caller
    exe = _build_c_caller(tmp_path)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "equal to the oracle" in out.stdout
