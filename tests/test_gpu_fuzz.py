"""Randomised parity: 24 seeded random cases of tools/fuzz_tc.py (database size and
subspace split, data kind, N, frames, tc_k, CTA pairs, chunking, seeding, path), each
bit-identical to the oracle.  The same tool ran 1,102 cases (20 minutes) in round 1."""
import os
import sys

import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
import fuzz_tc  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", [11, 12, 13])
def test_fuzz_bit_exact(seed):
    assert fuzz_tc.run(secs=600, seed=seed, max_cases=8) == 8
