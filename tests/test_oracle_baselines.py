"""The oracle's restatement of the comparison methods (baselines.py:36-154)
and concordant_fraction (cli.py:349-386) against golden vectors produced by
running the reference itself (tests/golden/make_baselines_golden.py).
Foster, CG and concordant_fraction reproduce bit for bit (same matvec, same
numpy reductions); the dense solve to LAPACK rounding."""
from __future__ import annotations

import json
import os

import numpy as np
import pytest

from oracle import katz_oracle as O

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def bl():
    with open(os.path.join(GOLDEN, "baselines.json")) as fh:
        idx = json.load(fh)
    return idx, np.load(os.path.join(GOLDEN, "baselines_cases.npz"))


def oracle_graph(arr, name):
    e = arr[f"{name}/edges"]
    n = {"star6": 6, "star50": 50, "grid5x6": 30, "grid7x7": 49, "grid8x8": 64, "cycle4": 4,
         "k5": 5, "edgeless3": 3, "edgeless4": 4, "dpath3": 3, "der3": 40}.get(name)
    if n is None:
        n = int(name[2:4])
    return O.CSRGraph.from_edges(n, e)


def run_oracle(method, g, kw):
    fn = {"foster": O.foster, "cg": O.cg_katz, "dense": O.dense_oracle}[method]
    try:
        return "ok", fn(g, **kw)
    except O.OracleBaselineError as e:
        return e.kind, e.partial


def test_oracle_baselines_match_reference(bl):
    idx, arr = bl
    for c in idx["cases"]:
        g = oracle_graph(arr, c["graph"])
        status, sv = run_oracle(c["method"], g, c["kwargs"])
        assert status == c["status"], c
        if sv is None:
            continue
        ref = arr[f"{c['key']}/values"]
        if c["method"] == "dense":
            np.testing.assert_allclose(sv.values, ref, rtol=1e-13, atol=1e-15)
        else:
            np.testing.assert_array_equal(sv.values, ref)
            assert sv.iterations == c["iterations"]
            assert sv.residual == c["residual"]
            np.testing.assert_array_equal(sv.ranking(), arr[f"{c['key']}/ranking"])


def test_oracle_concordant_fraction(bl):
    idx, arr = bl
    for c in idx["concordant"]:
        a, b, cc = (arr[f"{c['key']}/{x}"] for x in "abc")
        assert O.concordant_fraction(a, b) == c["ab"]
        assert O.concordant_fraction(a, cc) == c["ac"]
        assert O.concordant_fraction(a, a) == c["aa"]
