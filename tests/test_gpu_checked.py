"""The bounds-checked library (OL_LIB=checked: every kernel's index arithmetic checked on the
device, the stand-in for compute-sanitizer memcheck, which this pool does not run) with
poisoned buffers (OL_POISON=1: padding rows and coords NaN bytes, per-query outputs filled
with garbage first -- the initcheck stand-in) over tools/sanitize_cases.py: every kernel
reached, every result still equal to the oracle, zero failed device checks."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_checked_library_poisoned_cases():
    env = dict(os.environ, OL_LIB="checked", OL_POISON="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_cases.py"), "4"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert "CHECKED (device bounds checks: 0 failures)" in out and "poison on" in out, out[-2000:]
