"""Pins for the oracle's feature and distance (CPU only).

Each pin is external to the oracle: a closed form, numpy's
FFT (an independent library algorithm vs the oracle's direct summation), the
DFT shift theorem, or an exact rational emulation of the fp32 fmaf chain.
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


# ---------------------------------------------------------------- feature
def test_constant_profile_is_degenerate():
    c, deg = oracle.extract_feature(np.full(128, 0.7))
    assert deg and np.all(c == 0.0)


def test_single_tone_is_e1():
    W = 128
    p = np.cos(2 * np.pi * np.arange(W) / W)
    c, deg = oracle.extract_feature(p)
    assert not deg
    e1 = np.zeros(64); e1[0] = 1.0
    assert np.max(np.abs(c - e1)) < 1e-12


def test_pure_tone_k_maps_to_bin_k():
    W = 256
    for k in (2, 7, 33, 64):
        p = 0.3 + np.sin(2 * np.pi * k * np.arange(W) / W + 0.4)
        c, _ = oracle.extract_feature(p)
        assert abs(c[k - 1] - 1.0) < 1e-12 and np.max(np.abs(np.delete(c, k - 1))) < 1e-10


@pytest.mark.parametrize("seed", range(10))
def test_matches_numpy_fft(seed):                      # S:59 (library FFT, not the oracle's algorithm)
    rng = np.random.default_rng(seed)
    p = rng.random(256)
    c, deg = oracle.extract_feature(p)
    m = np.abs(np.fft.fft(p))[1:65]
    assert not deg
    assert np.max(np.abs(c - m / np.linalg.norm(m))) < 1e-9


@pytest.mark.parametrize("seed", range(10))
def test_rotation_brightness_scale_invariance(seed):
    rng = np.random.default_rng(100 + seed)
    p = rng.random(256)
    c0, _ = oracle.extract_feature(p)
    for s in rng.integers(1, 256, 4):
        c, _ = oracle.extract_feature(np.roll(p, int(s)))
        assert np.max(np.abs(c - c0)) < 1e-9
    c, _ = oracle.extract_feature(p + 3.25)
    assert np.max(np.abs(c - c0)) < 1e-9
    c, _ = oracle.extract_feature(p * 7.5)
    assert np.max(np.abs(c - c0)) < 1e-9
    assert abs(np.linalg.norm(c0) - 1.0) < 1e-9 and np.all(c0 >= 0)


# ---------------------------------------------------------------- distance chain (R3)
def _rn32(fr: Fraction) -> np.float32:
    """Correctly rounded (nearest, ties-to-even) binary32 of an exact rational."""
    x = np.float32(float(fr))
    cands = {np.nextafter(x, np.float32(-np.inf)), x, np.nextafter(x, np.float32(np.inf))}

    def rank(c):
        return (abs(Fraction(float(c)) - fr), int(np.float32(c).view(np.uint32)) & 1)
    return np.float32(min(cands, key=rank))


def _acc_exact_emulation(q, f) -> np.float32:
    acc = np.float32(0.0)
    for a, b in zip(q, f):
        d = _rn32(Fraction(float(a)) - Fraction(float(b)))
        acc = _rn32(Fraction(float(d)) ** 2 + Fraction(float(acc)))
    return acc


def test_acc_bit_exact_vs_rational_emulation():
    rng = np.random.default_rng(7)
    for trial in range(60):
        K = 64
        q = rng.random(K).astype(np.float32)
        f = rng.random(K).astype(np.float32)
        if trial % 3 == 1:
            f = (q + rng.standard_normal(K).astype(np.float32) * np.float32(1e-4)).astype(np.float32)
        if trial % 3 == 2:
            q = (q / np.linalg.norm(q)).astype(np.float32) * np.float32(1e-3)
            f = (f / np.linalg.norm(f)).astype(np.float32) * np.float32(1e-3)
        a = oracle.acc(q, f)
        e = _acc_exact_emulation(q, f)
        assert a.view(np.uint32) == e.view(np.uint32), (trial, a, e)


def test_distance_closed_forms():
    g = json.load(open(os.path.join(GOLD, "spec_examples.json")))["orthonormal_distance"]
    rng = np.random.default_rng(1)
    f = rng.random(64).astype(np.float32)
    a = oracle.acc(f, f)
    assert a == 0.0 and not np.signbit(a)
    e0 = np.zeros(64, np.float32); e0[0] = 1
    e1 = np.zeros(64, np.float32); e1[1] = 1
    assert oracle.acc(e0, e1) == np.float32(g["acc"])
    assert int(oracle.distance(e0, e1).view(np.uint32)) == int(g["dist_bits"], 16)
    assert oracle.distance(e0, e1) == np.sqrt(np.float32(2.0))


def test_acc_within_recursive_sum_bound_of_binary64():
    # |acc32 - acc64| <= (K+2) 2^-24 acc64 for non-negative terms
    rng = np.random.default_rng(3)
    K = 64
    F = np.abs(rng.standard_normal((2000, K))).astype(np.float32)
    F /= np.linalg.norm(F, axis=1, keepdims=True)
    q = F[0] * np.float32(0.9) + F[1] * np.float32(0.1)
    q = (q / np.linalg.norm(q)).astype(np.float32)
    a32 = oracle.acc_many(q, F).astype(np.float64)
    a64 = ((q.astype(np.float64)[None, :] - F.astype(np.float64)) ** 2).sum(1)
    assert np.all(np.abs(a32 - a64) <= (K + 2) * 2.0 ** -24 * a64 + 1e-45)


def test_acc_many_equals_acc():
    rng = np.random.default_rng(4)
    F = rng.random((300, 64)).astype(np.float32)
    q = rng.random(64).astype(np.float32)
    a = oracle.acc_many(q, F)
    for t in range(0, 300, 17):
        assert a[t].view(np.uint32) == oracle.acc(q, F[t]).view(np.uint32)


# ---------------------------------------------------------------- shift distance (NEXT-1)
def test_shift_distance_recovers_rotation():
    rng = np.random.default_rng(5)
    d = rng.random(256).astype(np.float32)
    for s0 in (0, 1, 37, 219, 255):
        q = np.roll(d, s0)          # q[(w + s0) mod W] == d[w]
        v, s = oracle.shift_distance(q, d)
        assert v == 0.0 and s == s0


def test_shift_distance_brute_force_and_exact_chain():
    rng = np.random.default_rng(6)
    for _ in range(4):
        q = rng.random(64).astype(np.float32); d = rng.random(64).astype(np.float32)
        # every shift's value is the pinned fp32 chain (oracle.acc) of the rotated profile
        vals = [oracle.acc(np.roll(q, -s), d) for s in range(64)]
        v, s = oracle.shift_distance(q, d)
        assert v.view(np.uint32) == min(vals).view(np.uint32) and s == int(np.argmin(vals))
        # and within the binary64 bound of the exact shift distance
        v64 = min(float(np.sum((np.roll(q, -k).astype(np.float64) - d) ** 2)) for k in range(64))
        assert abs(float(v) - v64) <= 66 * 2.0 ** -24 * v64 + 1e-30


def test_shift_distance_ties_take_smallest_shift():
    q = np.full(32, 0.5, np.float32)
    v, s = oracle.shift_distance(q, q)
    assert v == 0.0 and s == 0
    p = np.tile(np.float32([0.1, 0.9]), 16)          # period 2: shifts 0, 2, 4 ... tie
    v, s = oracle.shift_distance(np.roll(p, 1), p)
    assert v == 0.0 and s == 1


# ---------------------------------------------------------------- NEXT-1 stored profile
def _profiles(seed, n=6, W=256):
    """Synthetic omnidirectional profiles: a few Gaussian bumps on an offset + noise."""
    rng = np.random.default_rng(seed)
    w = np.arange(W)
    out = []
    for _ in range(n):
        x = 0.5 + 0.02 * rng.standard_normal(W)
        for _ in range(int(rng.integers(3, 9))):
            c, a, s = rng.uniform(0, W), rng.uniform(0.1, 0.5), rng.uniform(2, 12)
            d = (w - c + W / 2) % W - W / 2
            x += a * np.exp(-0.5 * (d / s) ** 2)
        out.append(x)
    return np.array(out)


@pytest.mark.parametrize("seed", range(4))
def test_shift_profile_spectrum_is_the_descriptor(seed):          # S:53, SURVEY 8f NEXT-1
    """numpy.fft of the stored profile: zero mean (DC bin 0) and |X_k| bins 1..64 equal the
    descriptor (the oracle's own direct DFT feature) to 1e-12 -- the scaling is 1/||m||."""
    for x in _profiles(seed):
        p64, p32 = oracle.shift_profile(x)
        c, deg = oracle.extract_feature(x)
        assert not deg
        X = np.fft.fft(p64)
        assert abs(X[0]) < 1e-12
        assert np.max(np.abs(np.abs(X[1:65]) - c)) < 1e-12
        assert np.array_equal(p32, p64.astype(np.float32))


def test_shift_profile_invariances_and_degenerate():
    """Affine invariance (brightness offset, positive gain) and rotation equivariance of the
    stored profile; a constant profile is all zeros (degenerate)."""
    for x in _profiles(7):
        p, _ = oracle.shift_profile(x)
        q, _ = oracle.shift_profile(3.5 * x + 0.7)
        assert np.max(np.abs(p - q)) < 1e-12
        r, _ = oracle.shift_profile(np.roll(x, 37))
        assert np.max(np.abs(r - np.roll(p, 37))) < 1e-12
    z64, z32 = oracle.shift_profile(np.full(256, 0.42))
    assert not z64.any() and not z32.any()


@pytest.mark.parametrize("seed", range(3))
def test_shift_distance_lower_bounded_by_descriptor_distance(seed):   # Parseval, SURVEY 8f NEXT-1
    """For every pair of stored profiles and EVERY circular shift s, the binary64 profile
    distance is >= (2/W) ||c_q - c_d||^2 (Parseval + the reverse triangle inequality on bins
    k and W-k); checked by brute force over all 256 shifts, and the bound is not vacuous."""
    P = _profiles(100 + seed, n=8)
    W = P.shape[1]
    prof = [oracle.shift_profile(x)[0] for x in P]
    desc = [oracle.extract_feature(x)[0] for x in P]
    ratios = []
    for i in range(len(P)):
        for j in range(len(P)):
            lb = (2.0 / W) * np.sum((desc[i] - desc[j]) ** 2)
            d = np.array([np.sum((np.roll(prof[i], -s) - prof[j]) ** 2) for s in range(W)])
            assert np.all(d >= lb * (1 - 1e-12) - 1e-15), (i, j, d.min(), lb)
            if i != j:
                ratios.append(lb / d.min())
    assert max(ratios) > 0.05     # the descriptor distance is a real (not trivial) bound
