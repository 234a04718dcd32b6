"""The checked build (make -C paper_1807_03847_b200/csrc checked): device
invariants (KB_DCHECK: indices in range, counts within capacity) are
counted on the device and polled after every C-ABI call -- the stand-in
for compute-sanitizer, which is closed on the GPU pool.
tools/checked_suite.sh runs the whole -m gpu suite with KB_LIB=checked."""
from __future__ import annotations

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHECKED = os.path.join(ROOT, "paper_1807_03847_b200", "_lib_checked", "libkatzb200.so")

PROBE = r"""
import ctypes, sys
sys.path.insert(0, %r)
from paper_1807_03847_b200 import _lib
L = _lib.lib()
assert "_lib_checked" in _lib.LIB_PATH
assert L.kb_sync(0) == 0                      # nothing failed yet
L.kb_tune(b"dcheck.selftest", 1)
rc = L.kb_sync(0)
msg = _lib.last_error()
L.kb_tune(b"dcheck.selftest", 0)
assert rc == _lib.KB_ECUDA and "KB_DCHECK failed" in msg and "kb_api.cu" in msg, (rc, msg)
assert L.kb_sync(0) == 0                      # reported once, then re-armed
print("ok")
""" % ROOT


def test_checked_build_reports_device_invariant_failures():
    if not os.path.exists(CHECKED):
        pytest.skip("checked build missing (make -C paper_1807_03847_b200/csrc checked)")
    out = subprocess.run([sys.executable, "-c", PROBE], capture_output=True, text=True,
                         timeout=300, env=dict(os.environ, KB_LIB="checked"))
    assert out.returncode == 0 and out.stdout.strip().endswith("ok"), out.stderr[-2000:]
