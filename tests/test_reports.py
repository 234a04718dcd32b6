"""Report serialization (reports.py restated) against the reference's own
output (tests/golden/baselines.json 'samples', from make_baselines_golden.py).
Host-only formatting: runs without a GPU."""
from __future__ import annotations

import json
import os

from paper_1807_03847_b200 import reports as R

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")

SAMPLE = {"a": 1.0, "b": 0.1, "c": -0.0, "d": float("nan"), "e": float("inf"),
          "f": 1e-300, "g": 123456789012345678, "h": [], "i": {}, "j": [1, 2.5, None, True],
          "k": {"x": "q\"uote", "y": [{"z": 3}]}, "l": 2.0 ** 70}


def _golden():
    with open(os.path.join(GOLDEN, "baselines.json")) as fh:
        return json.load(fh)


def test_json_and_floats_match_reference():
    s = _golden()["samples"]
    assert R.dumps_json(SAMPLE) == s["json"]
    assert R.dumps_json(SAMPLE, indent=4) == s["json4"]
    assert [R.format_float(x) for x in (1.0, 0.1, 1e22, 1e-7, 123.0, 2.0 ** 60)] == s["floats"]


def test_run_report_layout_and_csv_roundtrip():
    rep = R.RunReport(command="static", method="katz-bounds", parameters={"alpha": 0.25},
                      iterations=3, wall_time_s=0.5, separated_fraction=0.75,
                      ranking_prefix=[2, 0], extra={"note": "x"})
    d = rep.to_dict()
    assert list(d) == ["command", "method", "parameters", "iterations", "wall_time_s",
                       "separated_fraction", "ranking_prefix", "note"]
    rows = R.node_rows([2, 0, 1], [0.5, 0.25, 1.0], [0.6, 0.3, 1.5], cap=2)
    assert rows == [dict(node_id=2, lower=1.0, upper=1.5, rank=1),
                    dict(node_id=0, lower=0.5, upper=0.6, rank=2)]
    assert R.dumps_csv(rows) == "node_id,lower,upper,rank\n2,1.0,1.5,1\n0,0.5,0.59999999999999998,2\n"
    # every golden CSV re-serialises to itself through the float formatter
    for rep in _golden()["reports"]:
        lines = rep["static_csv"].splitlines()
        assert lines[0] == ",".join(R.CSV_COLUMNS)
        rows = []
        for ln in lines[1:]:
            a, lo, up, rk = ln.split(",")
            rows.append(dict(node_id=int(a), lower=float(lo), upper=float(up), rank=int(rk)))
        assert R.dumps_csv(rows) == rep["static_csv"]
