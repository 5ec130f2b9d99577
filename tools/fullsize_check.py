"""Full-size sampled parity at BASELINE's C4 (100M rows, 1,024 frames, the bench's launch
configuration), with more sampled frames than tests/test_gpu_fullsize.py: the oracle
recomputes each sampled frame against the entire database.
usage: python tools/fullsize_check.py [n_samples] [config]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
from test_gpu_fullsize import _sampled_parity  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 16
cfg = sys.argv[2] if len(sys.argv) > 2 else "C4"
sample = sorted(set(int(x) for x in np.random.default_rng(2024).choice(1024, n, replace=False)))
e = _sampled_parity(cfg, sample)
print(f"{cfg}: {len(sample)} sampled frames bit-exact (candidates and estimates) vs the oracle over the full "
      f"database; tc_k {e.stat('tc_k')}, pairs {e.stat('used_pair')}, survivors/pair {e.stat('survivors') / e.stat('pairs'):.2e}")
