"""NEXT-3 parity: GPU descriptor extraction (extract_kernel, P:121 / S:53) vs the
oracle's binary64 direct-summation DFT feature.

Tolerances: both sides compute the same binary64 definition with different
summation orders (the norm is a warp reduction on the GPU, a running sum in the
oracle), so binary64 values agree to a few ulps of 1 (checked at 1e-13); the fp32
descriptor is RN32 of the binary64 value on both sides, so it is bit-identical
except where the binary64 value sits within those few ulps of an fp32 rounding
boundary (checked: at most 1 fp32 ulp, and bit-identical for >= 99 % of values).
The degenerate decision (||m|| <= 1e-12) is taken in binary64 on both sides."""
import numpy as np
import pytest
import torch

import oracle
import synthgen
import paper_2006_08861_b200 as ol

pytestmark = pytest.mark.gpu


def _oracle(P):
    d = np.zeros((P.shape[0], 64))
    g = np.zeros(P.shape[0], bool)
    for i, p in enumerate(P):
        d[i], g[i] = oracle.extract_feature(p)
    return d, g


def _check(P, o32, deg, o64):
    ref, rdeg = _oracle(P)
    assert np.array_equal(deg, rdeg)
    assert np.max(np.abs(o64 - ref)) <= 1e-13, np.max(np.abs(o64 - ref))
    r32 = ref.astype(np.float32)
    ulp = np.abs(o32.view(np.int32).astype(np.int64) - r32.view(np.int32).astype(np.int64))
    assert ulp.max() <= 1
    assert (ulp == 0).mean() >= 0.99


@pytest.mark.parametrize("W", [256, 128, 65, 1000, 2048])
def test_extract_random_profiles_vs_oracle(W):
    rng = np.random.default_rng(W)
    n = 300 if W <= 1000 else 40           # several CTAs (8 profiles each) + a ragged tail
    P = rng.random((n, W)) + np.sin(np.arange(W) * 2 * np.pi * 3 / W)[None, :] * rng.random((n, 1))
    P[3] = 0.7                             # constant -> degenerate
    P[5] = 0.0
    e = ol.Engine(0)
    o32, deg, o64 = e.extract_features(P, want64=True)
    assert deg[3] and deg[5] and not deg[0]
    assert np.all(o32[3] == 0) and np.all(o64[5] == 0)
    _check(P, o32, deg, o64)


def test_extract_device_path_equals_host_path():
    rng = np.random.default_rng(7)
    P = rng.random((1000, 256))
    e = ol.Engine(0)
    h32, hdeg, h64 = e.extract_features(P, want64=True)
    d32, ddeg, d64 = e.extract_features(torch.from_numpy(P).cuda(), want64=True)
    torch.cuda.synchronize()
    assert np.array_equal(h32.view(np.uint32), d32.cpu().numpy().view(np.uint32))
    assert np.array_equal(h64.view(np.uint64), d64.cpu().numpy().view(np.uint64))
    assert np.array_equal(hdeg, ddeg.cpu().numpy())


def test_extract_generator_profiles_give_the_database_descriptors():
    # the generator's own descriptors are RN32 of the same binary64 definition
    spec = synthgen.Spec(seed=51, n_floors=1, paths=2, frames_per_path=150)
    pts = synthgen.entry_points(spec, 0, spec.n_entries)
    r = synthgen.render_host(spec, pts, profiles=True, f64=True)
    e = ol.Engine(0)
    o32, deg, o64 = e.extract_features(r["profile"], want64=True)
    assert not deg.any()
    assert np.max(np.abs(o64 - r["desc64"])) <= 1e-13
    ulp = np.abs(o32.view(np.int32).astype(np.int64) - r["desc"].view(np.int32).astype(np.int64))
    assert ulp.max() <= 1 and (ulp == 0).mean() >= 0.99
    _check(r["profile"], o32, deg, o64)


def test_extract_rotation_brightness_scale_invariance():   # P:121 "rotation-invariant"
    rng = np.random.default_rng(9)
    p = rng.random(256)
    P = np.stack([p, np.roll(p, 37), np.roll(p, 255), p + 3.25, p * 7.5])
    e = ol.Engine(0)
    _, _, o64 = e.extract_features(P, want64=True)
    assert np.max(np.abs(o64 - o64[0])) <= 1e-12


def test_extracted_query_retrieves_its_own_rotated_entry():   # the path fed by NK9
    spec = synthgen.Spec(seed=52, n_floors=1, paths=1, frames_per_path=400)
    pts = synthgen.entry_points(spec, 0, spec.n_entries)
    r = synthgen.render_host(spec, pts, profiles=True)
    e = ol.Engine(0)
    F, deg = e.extract_features(r["profile"])
    rows = np.array([0, 17, 250, 399])
    Q, _ = e.extract_features(np.stack([np.roll(r["profile"][i], 91) for i in rows]))
    e.upload(F, r["tiles"], [F.shape[0]], spec.grid())
    e.query(Q[:, None, :], N=3, aggregate=False)
    c = e.topk()
    ref = oracle.retrieve([F.shape[0]], F, r["tiles"], Q[:, None, :], 3)
    assert np.array_equal(c["frame"], ref.frame)
    assert np.array_equal(c["dist2"].view(np.uint32), ref.acc.view(np.uint32))


def test_extract_argument_errors():
    e = ol.Engine(0)
    with pytest.raises(ol.OmnilocError):
        e.extract_features(np.zeros((4, 64)))            # W must exceed K = 64
    with pytest.raises(ol.OmnilocError):
        e.extract_features(np.zeros((4, 2049)))          # shared-memory bound
    with pytest.raises(ol.OmnilocError):
        e.extract_features(np.full((2, 256), np.nan))    # S:32 finite values
    o32, deg = e.extract_features(np.zeros((0, 256)))
    assert o32.shape == (0, 64) and deg.shape == (0,)


@pytest.mark.parametrize("W", [128, 256, 512, 1000])
def test_stored_profiles_vs_oracle(W):                       # NEXT-1 stored profile
    """(x - mean x)/||m|| from the extraction kernels (FFT path for 128/256/512, direct sum for
    1000) vs the oracle's binary64 definition rounded to fp32: <= 1 fp32 ulp, >= 99 %
    bit-identical; degenerate profiles give zeros."""
    rng = np.random.default_rng(W + 1)
    P = rng.random((160, W)) + np.cos(np.arange(W) * 2 * np.pi * 5 / W)[None, :] * rng.random((160, 1))
    P[7] = 1.25
    e = ol.Engine(0)
    o32, deg, po = e.extract_features(P, want_profiles=True)
    assert po.shape == (160, W) and deg[7] and not po[7].any()
    ref = np.stack([oracle.shift_profile(x)[1] for x in P])
    ulp = np.abs(po.view(np.int32).astype(np.int64) - ref.view(np.int32).astype(np.int64))
    assert ulp.max() <= 1, ulp.max()
    assert (ulp == 0).mean() >= 0.99
    # device input: same values
    o32d, degd, pod = e.extract_features(torch.from_numpy(P).cuda(), want_profiles=True)
    torch.cuda.synchronize()
    assert np.array_equal(pod.cpu().numpy(), po) and np.array_equal(o32d.cpu().numpy(), o32)


@pytest.mark.parametrize("n", [1, 2, 9, 301])
def test_extract_w256_pairs_odd_counts_and_scale_disparity(n):
    """W = 256 runs two profiles per warp as one complex transform: odd counts leave a lone
    profile, and a pair may mix profiles of very different brightness (scales 1e-4 and 3e5
    apart; each is scaled by a power of two first) -- each must still match the oracle."""
    rng = np.random.default_rng(1000 + n)
    W = 256
    P = rng.random((n, W)) + np.sin(np.arange(W) * 2 * np.pi * 7 / W)[None, :] * rng.random((n, 1))
    if n >= 2:
        P[1] *= 1e-4                                   # pair (0, 1): magnitudes 1e-4 apart
    if n >= 9:
        P[8] *= 3e5                                    # bright, lone when n = 9
        P[3] = 0.0                                     # degenerate partner of profile 2
    e = ol.Engine(0)
    o32, deg, o64 = e.extract_features(P, want64=True)
    _check(P, o32, deg, o64)
    _, _, po = e.extract_features(P, want_profiles=True)
    ref = np.stack([oracle.shift_profile(x)[1] for x in P])
    ulp = np.abs(po.view(np.int32).astype(np.int64) - ref.view(np.int32).astype(np.int64))
    assert ulp.max() <= 1, ulp.max()
