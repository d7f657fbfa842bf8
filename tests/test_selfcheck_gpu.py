"""Self-check runs (SURVEY §4 test layer 5; compute-sanitizer is closed on the
GPU pool): every kernel family -- the fused last-CTA finalize, K1, the
look-back scan, the wide / grouped finalize, the sparse grouping, pack and
merge, the library-owned exchange with its capacity retry, prepared graphs --
through the self-check build (device checks of index and protocol invariants,
-DHD_CHECKS) repeated with bit-identical outputs each time and nothing written
past the reported children."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_self_check_build_stress():
    from paper_1802_06215_b200 import build as B
    lib = B.build_checked()
    env = dict(os.environ, DESPOT_LIB=lib)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "sanitize_cases.py"), "--stress", "5"],
                         capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-3000:]
    assert "libdespot_checked.so" in out.stdout
    assert out.stdout.count(" ok x 5") == 7, out.stdout
