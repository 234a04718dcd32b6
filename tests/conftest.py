"""Test configuration: the `gpu` marker and shared fixtures.

`-m "not gpu"` runs here (no GPU): oracle vs golden vectors, host logic, the
C-ABI symbol table.  `-m gpu` runs on a B200 and compares the CUDA path with
the oracle through the C-ABI.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


@pytest.fixture(scope="session")
def golden_index():
    with open(os.path.join(GOLDEN, "digests.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def small_cases():
    return dict(np.load(os.path.join(GOLDEN, "small_cases.npz")))


@pytest.fixture(scope="session")
def dynamic_cases():
    return dict(np.load(os.path.join(GOLDEN, "dynamic_cases.npz")))
