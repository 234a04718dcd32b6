"""pytest plugin (test infrastructure): makes ``import katzbounds`` resolve to
this package, so the reference's own test suite (installed unmodified in
baseline/_ref/katzbounds_tests by tools/install_reference.sh) runs against
the B200 implementation.  Loaded with ``-p tests.ref_alias_plugin``."""
from __future__ import annotations

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
# the real reference must not be importable in this process
sys.path[:] = [p for p in sys.path if os.path.abspath(p or ".") != REF]
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import paper_1807_03847_b200 as _pkg  # noqa: E402
from paper_1807_03847_b200 import reports as _reports  # noqa: E402

sys.modules["katzbounds"] = _pkg
sys.modules["katzbounds.reports"] = _reports
