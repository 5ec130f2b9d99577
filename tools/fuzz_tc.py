"""Randomised GPU-vs-oracle stress of the scan paths.

Each case draws random values for:
- database size and subspace split, and the data kind;
- N, the frame count and bundle size M;
- tc_k, CTA pairs, chunk size and seeding;
- the path (tensor-core or CUDA-core), and whether Algorithm 2 runs.

Every case must be bit-identical to the oracle.
usage: python tools/fuzz_tc.py [seconds] [seed]   (tests/test_gpu_fuzz.py runs a few cases)"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)
import oracle  # noqa: E402
import synthgen  # noqa: E402
import paper_2006_08861_b200 as ol  # noqa: E402
from gpu_helpers import assert_candidates_equal, assert_estimates_equal  # noqa: E402


def one_case(rng, idx):
    kind = rng.choice(["paper", "signed", "flat", "dup"])
    rows = int(rng.integers(300, 60000))
    if kind == "paper":
        spec = synthgen.Spec(seed=int(rng.integers(1, 10**6)), n_floors=int(rng.integers(1, 4)), paths=5,
                             frames_per_path=max(20, rows // 15))
        F, C = synthgen.db_host(spec)
        rows = F.shape[0]
        Qall = synthgen.render_host(spec, synthgen.query_points(spec, int(rng.integers(1, 10**6)), 800))["desc"]
    else:
        if kind == "flat":
            F = synthgen.gflat(rows, seed=int(rng.integers(1, 10**6)), dup_frac=0.05)
        else:
            F = (rng.standard_normal((rows, 64)) * rng.choice([0.01, 1.0, 5.0])).astype(np.float32)
            if kind == "dup":
                F[rng.integers(0, rows, rows // 5)] = F[rng.integers(0, rows, rows // 5)]
        C = rng.integers(0, 4000, (rows, 2)).astype(np.int32)
        Qall = F[rng.integers(0, rows, 800)] + (rng.standard_normal((800, 64)) * 1e-3).astype(np.float32)
    ns = int(rng.integers(1, 5))
    cuts = np.sort(rng.choice(np.arange(1, rows), ns - 1, replace=False)) if ns > 1 else np.array([], int)
    sizes = [int(x) for x in np.diff(np.concatenate([[0], cuts, [rows]]))]
    M = int(rng.choice([1, 1, 3, 5]))
    B = int(rng.integers(2, 700 // M + 1))
    Q = np.ascontiguousarray(Qall[:B * M].reshape(B, M, 64))
    N = int(rng.choice([1, 5, 15, 15, 33, 64]))
    opts = {"tc": 1, "tc_k": int(rng.choice([32, 64, 0])), "pair": int(rng.choice([0, 1, 2]))}
    if rng.random() < 0.3:
        opts["chunk"] = int(rng.choice([4096, 8192, 50000]))
    if rng.random() < 0.2:
        opts["tau_seed"] = 0
    if rng.random() < 0.15:
        opts["tc"] = 0
    # schedule / kernel-choice options (results never depend on them)
    if rng.random() < 0.25:
        opts["seed_kernel"] = int(rng.choice([0, 1]))
    if rng.random() < 0.25:
        opts["seed_samples"] = int(rng.choice([16, 300, 4096, 20000]))
    if rng.random() < 0.2:
        opts["cluster"] = int(rng.choice([2, 4]))
    if rng.random() < 0.15:
        opts["ctas"] = int(rng.choice([1, 37]))
    if rng.random() < 0.2:
        opts["scan2"] = int(rng.choice([0, 1, 2]))
    if rng.random() < 0.15:
        opts["tc_min_frames"] = int(rng.choice([1, 64, 100000]))
        opts["tc"] = -1
    if rng.random() < 0.15:
        opts["merge_scan"] = 1
    if rng.random() < 0.15:
        opts["agg_block"] = 1
    if rng.random() < 0.5:
        opts["inline_rescore"] = int(rng.choice([0, 1]))
    e = ol.Engine(0, coarse_k=16)
    if os.environ.get("OL_POISON") == "1":
        e.set_option("poison", 1)
    for k, v in opts.items():
        e.set_option(k, v)
    e.upload(F, C, sizes, (4096, 4096))
    agg = bool(rng.random() < 0.5)
    e.query(Q, N=N, aggregate=agg)
    ref = oracle.retrieve(sizes, F, C, Q, N)
    ctx = f"case {idx}: {kind} rows={rows} sizes={sizes} B={B} M={M} N={N} agg={agg} {opts}"
    assert_candidates_equal(e.topk(), ref, ctx)
    if agg:
        assert_estimates_equal(e.estimates(), ref, ctx=ctx)
    e.close()


def run(secs=300.0, seed=1, max_cases=None):
    rng = np.random.default_rng(seed)
    t_end = time.time() + secs
    cases = 0
    while time.time() < t_end and (max_cases is None or cases < max_cases):
        one_case(rng, cases)
        cases += 1
    return cases


if __name__ == "__main__":
    n = run(float(sys.argv[1]) if len(sys.argv) > 1 else 300, int(sys.argv[2]) if len(sys.argv) > 2 else 1)
    print(f"fuzz ok: {n} cases bit-exact vs the oracle")
