"""The shared input generator (synthgen) produces what DESIGN.md §4 says:
descriptors equal to the oracle's own feature extraction of the rendered
profile, unit norm, rotation-invariant, paper-shaped spectra, and
shard-independent draws.  CPU only."""
import dataclasses

import numpy as np

import oracle
import synthgen


def test_descriptor_is_oracle_feature_of_profile():
    spec = synthgen.Spec(seed=11, n_floors=2, paths=2, frames_per_path=30)
    pts = synthgen.entry_points(spec, 0, spec.n_entries)[::7]
    r = synthgen.render_host(spec, pts, profiles=True, f64=True)
    for i in range(len(pts)):
        c, deg = oracle.extract_feature(r["profile"][i], 64)
        assert not deg
        assert np.max(np.abs(c - r["desc64"][i])) < 1e-9
        assert np.array_equal(r["desc"][i], r["desc64"][i].astype(np.float32))


def test_heading_is_a_rotation():
    spec = synthgen.Spec(seed=12, n_floors=1, paths=1, frames_per_path=10, noise_sigma=0.0)
    p = synthgen.entry_points(spec, 0, 1)
    q = p.copy()
    q["heading"] = p["heading"] + 2 * np.pi * 37 / spec.W
    a = synthgen.render_host(spec, p, profiles=True, f64=True)
    b = synthgen.render_host(spec, q, profiles=True, f64=True)
    assert np.max(np.abs(np.roll(a["profile"][0], -37) - b["profile"][0])) < 1e-9
    assert np.max(np.abs(a["desc64"][0] - b["desc64"][0])) < 1e-9


def test_shards_generate_independently_and_deterministically():
    spec = synthgen.Spec(seed=13, n_floors=1, paths=5, frames_per_path=40)
    F, C = synthgen.db_host(spec)
    F2, C2 = synthgen.db_host(spec, 77, 50)
    assert np.array_equal(F[77:127], F2) and np.array_equal(C[77:127], C2)
    F3, _ = synthgen.db_host(spec)
    assert np.array_equal(F, F3)


def test_paper_shaped_spectrum_and_tiles():
    spec = synthgen.CONFIGS["C2"].spec
    spec = dataclasses.replace(spec, frames_per_path=200)
    F, C = synthgen.db_host(spec)
    n = np.linalg.norm(F.astype(np.float64), axis=1)
    assert np.all(np.abs(n - 1) < 1e-6) and np.all(F >= 0)
    e = (F.astype(np.float64) ** 2)
    assert e[:, :16].sum(1).mean() > 0.97          # ~99 % in bins 1-16
    gw, gh = spec.grid()
    assert C[:, 0].min() >= 0 and C[:, 0].max() < gw and C[:, 1].min() >= 0 and C[:, 1].max() < gh
    assert sorted(set(C[:, 1].tolist())) == [20, 35, 50, 65, 80]     # 5 paths
