"""Golden vectors for the comparison methods (foster, cg_katz, dense_oracle)
and concordant_fraction, produced by running the *reference* here:

    python tests/golden/make_baselines_golden.py

Writes tests/golden/baselines_cases.npz and baselines.json (reference
baselines.py:36-154, cli.py:349-386).  Nothing at test time reads
/root/reference.
"""
from __future__ import annotations

import json
import os
import sys

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")

import numpy as np  # noqa: E402

import katzbounds as K  # noqa: E402
import builders  # noqa: E402
from katzbounds import baselines as B  # noqa: E402
from katzbounds.cli import concordant_fraction  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def edges_of(g):
    return np.array(sorted(g.arcs()), dtype=np.int64).reshape(-1, 2)


def graphs():
    out = [
        ("star6", builders.star(6)),
        ("star50", builders.star(50)),
        ("grid5x6", builders.grid(5, 6)),
        ("grid7x7", builders.grid(7, 7)),
        ("grid8x8", builders.grid(8, 8)),
        ("cycle4", builders.cycle(4)),
        ("k5", builders.complete(5)),
        ("edgeless3", K.Graph.from_edges(3, [])),
        ("edgeless4", K.Graph.from_edges(4, [])),
        ("dpath3", K.Graph.from_edges(3, [(0, 1), (1, 2)])),
    ]
    for seed in range(5):
        out.append((f"er40_{seed}", builders.er_graph(40, 0.1, seed=seed)))
        out.append((f"er60_{seed}", builders.er_graph(60, 0.08, seed=seed)))
    out.append(("der3", builders.er_graph(40, 0.08, seed=53, undirected=False)))
    return out


def run(fn, *a, **k):
    """(status, ScoreVector | partial | None)"""
    try:
        return "ok", fn(*a, **k)
    except K.ConvergenceError as e:
        return "convergence", e.partial
    except K.NumericError:
        return "numeric", None
    except K.MethodNotApplicableError:
        return "not_applicable", None
    except K.ParameterError:
        return "parameter", None


def main():
    arrays = {}
    index = []
    G = dict(graphs())
    for name, g in G.items():
        arrays[f"{name}/edges"] = edges_of(g)
    cases = []
    for name, g in G.items():
        d = max(g.max_out_degree(), 1)
        for alpha in (None, 0.5 / d):
            cases.append(("foster", name, dict(alpha=alpha, tol=1e-13)))
            cases.append(("foster", name, dict(alpha=alpha, tol=1e-9)))
            cases.append(("cg", name, dict(alpha=alpha, residual_tol=1e-15)))
            cases.append(("cg", name, dict(alpha=alpha, residual_tol=1e-4)))
            cases.append(("dense", name, dict(alpha=alpha)))
    # truncated Foster rounds = the engine's partial sums (test_baselines.py:65-74)
    for r in range(1, 9):
        cases.append(("foster", "grid5x6", dict(alpha=0.15, tol=1e-300, max_iter=r)))
    cases.append(("cg", "grid8x8", dict(alpha=0.2, residual_tol=1e-15, max_iter=2)))
    cases.append(("cg", "dpath3", dict(alpha=0.3)))
    cases.append(("foster", "star6", dict(alpha=0.5)))
    for i, (method, name, kw) in enumerate(cases):
        g = G[name]
        fn = {"foster": B.foster, "cg": B.cg_katz, "dense": B.dense_oracle}[method]
        status, sv = run(fn, g, **kw)
        key = f"c{i}"
        rec = dict(key=key, method=method, graph=name, kwargs=kw, status=status)
        if sv is not None:
            arrays[f"{key}/values"] = np.asarray(sv.values)
            arrays[f"{key}/ranking"] = np.asarray(sv.ranking(), dtype=np.int64)
            rec.update(iterations=sv.iterations, residual=sv.residual)
        index.append(rec)
    # concordant_fraction (cli.py:349-360) on random permutation pairs
    rng = np.random.default_rng(11)
    conc = []
    for i, n in enumerate([1, 2, 3, 10, 100, 1000, 5000]):
        a = rng.permutation(n)
        b = rng.permutation(n)
        c = a.copy()
        if n > 3:
            c[: n // 3] = np.sort(c[: n // 3])
        arrays[f"conc{i}/a"] = a
        arrays[f"conc{i}/b"] = b
        arrays[f"conc{i}/c"] = c
        conc.append(dict(key=f"conc{i}", n=n, ab=concordant_fraction(a, b),
                         ac=concordant_fraction(a, c), aa=concordant_fraction(a, a)))
    # the compare command's JSON report and a static CSV, via the reference
    # CLI itself (cli.py:293-346, reports.py)
    import tempfile
    from katzbounds import cli
    from katzbounds import reports as R
    from katzbounds.graph import dumps_edge_list
    reports = []
    with tempfile.TemporaryDirectory() as tmp:
        for name in ("grid7x7", "er60_1", "star50"):
            g = G[name]
            path = os.path.join(tmp, f"{name}.txt")
            with open(path, "w") as fh:
                fh.write(dumps_edge_list(g.node_count, sorted(
                    (u, v) for u, v in g.arcs() if u < v)))
            out = os.path.join(tmp, f"{name}.json")
            assert cli.main(["compare", path, "--undirected", "--out-file", out]) == 0
            csv_out = os.path.join(tmp, f"{name}.csv")
            assert cli.main(["static", path, "--undirected", "--out", "csv",
                             "--out-file", csv_out]) == 0
            with open(out) as fh, open(csv_out) as fc:
                reports.append(dict(graph=name, n=g.node_count, compare_json=fh.read(),
                                    static_csv=fc.read()))
    sample = {"a": 1.0, "b": 0.1, "c": -0.0, "d": float("nan"), "e": float("inf"),
              "f": 1e-300, "g": 123456789012345678, "h": [], "i": {}, "j": [1, 2.5, None, True],
              "k": {"x": "q\"uote", "y": [{"z": 3}]}, "l": 2.0 ** 70}
    samples = dict(json=R.dumps_json(sample), json4=R.dumps_json(sample, indent=4),
                   floats=[R.format_float(x) for x in (1.0, 0.1, 1e22, 1e-7, 123.0, 2.0 ** 60)])
    np.savez_compressed(os.path.join(HERE, "baselines_cases.npz"), **arrays)
    with open(os.path.join(HERE, "baselines.json"), "w") as fh:
        json.dump(dict(cases=index, concordant=conc, reports=reports, samples=samples), fh,
                  indent=1)
    print("cases", len(index), "concordant", len(conc))


if __name__ == "__main__":
    main()
