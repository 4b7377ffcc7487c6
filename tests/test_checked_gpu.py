"""The bounds-checked build on the GPU: tests/sanitize_run.py (every kernel of the
library once, the 2.1M pipelined ewsjf_tick_host included) in a subprocess that
loads libewsjf_check.so (EWSJF_CHECKED=1, device EWSJF_CHECK sites compiled in;
a failed check traps and the driver exits non-zero).  compute-sanitizer is not
available on the GPU pool; this is its stand-in."""
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "paper_2601_21758_b200", "libewsjf_check.so")


@pytest.mark.gpu
def test_sanitize_driver_under_bounds_checks():
    if not os.path.exists(CHECKED):
        pytest.skip("libewsjf_check.so not built (EWSJF_CHECKED=1 python -m paper_2601_21758_b200._build)")
    env = dict(os.environ, EWSJF_CHECKED="1", SANITIZE_BIG="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "sanitize_run.py")], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "sanitize driver done" in r.stdout, (r.stdout[-2000:], r.stderr[-2000:])
    assert "EWSJF_CHECK failed" not in r.stdout
