"""Full-size sampled parity (BASELINE.json configs C3 and C4, in the launch
configuration bench.py times): the GPU answers all 1,024 query frames; the
oracle recomputes a sample of them against the ENTIRE database (streamed to the
host in slices; every row's acc is independent, so slicing changes nothing) and
the results must match bit-for-bit, estimates included."""
import numpy as np
import pytest
import torch

import oracle
import synthgen
import paper_2006_08861_b200 as ol
from gpu_helpers import assert_candidates_equal, assert_estimates_equal

pytestmark = pytest.mark.gpu


def near_tie_frames(e, Qd, N, k):
    """The k query frames whose N-th and (N+1)-th best squared distances are closest (relative
    gap), found with one extra top-(N+1) query: where a wrong prune or a wrong tie order would
    show first (P:202 top N).  Only picks which frames to check; expected values come from
    the oracle."""
    e.query(Qd.view(-1, 1, 64), N=N + 1, aggregate=False)
    g = e.topk()["dist2"].reshape(-1, N + 1).astype(np.float64)
    gap = (g[:, N] - g[:, N - 1]) / np.maximum(g[:, N - 1], 1e-30)
    return [int(i) for i in np.argsort(gap, kind="stable")[:k]]


def _sampled_parity(name, sample, kc=16, near_ties=0):
    cfg = synthgen.CONFIGS[name]
    spec = cfg.spec
    n = spec.n_entries
    dev = torch.device("cuda", 0)
    F, C = synthgen.db_device(spec, 0, n, dev)
    Qd, _ = synthgen.render_device(spec, synthgen.query_points(spec, 4242, cfg.n_queries), dev)
    e = ol.Engine(0, coarse_k=kc)
    e.upload(F, C, [n], spec.grid())
    if near_ties:
        sample = sorted(set(sample) | set(near_tie_frames(e, Qd, cfg.N, near_ties)))
    e.query(Qd.view(-1, 1, 64), N=cfg.N, aggregate=True)
    got = e.topk()
    est = e.estimates()
    assert len(got) == cfg.n_queries * cfg.N
    Q = Qd.cpu().numpy()
    accs = [np.empty(n, np.float32) for _ in sample]
    step = 1 << 22
    for b in range(0, n, step):
        Fh = F[b:b + step].cpu().numpy()
        for j, q in enumerate(sample):
            accs[j][b:b + len(Fh)] = oracle.acc_many(Q[q], Fh)
    for j, q in enumerate(sample):
        idx, acc = oracle.topn(accs[j], cfg.N, "select")
        xy = C[torch.from_numpy(idx.astype(np.int64)).to(dev)].cpu().numpy()
        ref = oracle.Candidates(np.zeros(len(idx), np.uint32), idx, np.zeros(len(idx), np.uint32),
                                np.zeros(len(idx), np.uint32), acc, np.sqrt(acc),
                                xy[:, 0].copy(), xy[:, 1].copy())
        g = got[q * cfg.N:(q + 1) * cfg.N].copy()
        assert np.all(g["bundle"] == q)
        g["bundle"] = 0
        assert_candidates_equal(g, ref, f"{name} query {q}")
        assert_estimates_equal(est[q:q + 1], ref, ctx=f"{name} query {q}")
    return e


def test_c3_sampled():
    e = _sampled_parity("C3", [0, 1, 511, 1023])
    assert e.stat("survivors") < 0.05 * e.stat("pairs")


@pytest.mark.slow
def test_c4_sampled_bench_config():
    """C4 (100M rows) in the bench's launch configuration: 2 fixed frames plus the 8 frames
    with the smallest relative gap between their 15th and 16th best distances."""
    e = _sampled_parity("C4", [0, 777], near_ties=8)
    assert e.stat("used_tc") == 1
