"""The paper's method comparison at C2 scale on one B200 (Table 1 shape):
bounded Katz (top-100 and full ranking) next to Foster and CG on the same
device graph, plus the ranking agreement (concordant fraction) of each.

  python tools/compare_bench.py [--scale 24]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1807_03847_b200 as P  # noqa: E402
from paper_1807_03847_b200 import generators as G  # noqa: E402
from paper_1807_03847_b200.compare import ranking_inversions  # noqa: E402


def timed(fn):
    import torch
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = fn()
    torch.cuda.synchronize()
    return out, time.perf_counter() - t0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=24)
    ap.add_argument("--foster-tol", type=float, default=1e-9)
    ap.add_argument("--cg-tol", type=float, default=1e-15)
    a = ap.parse_args()
    g = G.rmat_graph(1 << a.scale, edge_factor=16, seed=42)
    n = g.node_count
    alpha = P.default_alpha(g)
    out = {"workload": f"rmat-s{a.scale}-ef16", "n": n, "nnz": g.arc_count, "alpha": alpha}
    # warm the device graph and the kernels once
    P.run(P.init(g, P.Criterion.top_k(100, 1e-6), undirected=True), g)
    res, t = timed(lambda: P.run(P.init(g, P.Criterion.top_k(100, 1e-6), undirected=True), g))
    out["katz_top100"] = {"s": t, "iterations": res.iterations_used}
    rk, t = timed(lambda: P.run(P.init(g, P.Criterion.ranking(1e-6), undirected=True), g))
    out["katz_ranking"] = {"s": t, "iterations": rk.iterations_used,
                           "separated_fraction": rk.separated_fraction}
    fo, t = timed(lambda: P.foster(g, alpha=alpha, tol=a.foster_tol))
    out["foster"] = {"s": t, "iterations": fo.iterations, "residual": fo.residual}
    cg, t = timed(lambda: P.cg_katz(g, alpha=alpha, residual_tol=a.cg_tol))
    out["cg"] = {"s": t, "iterations": cg.iterations, "residual": cg.residual}
    total = n * (n - 1) // 2
    for name, sv in (("foster", fo), ("cg", cg)):
        order_b, t_rank = timed(lambda: np.lexsort((np.arange(n), -sv.values)))
        inv, t = timed(lambda: ranking_inversions(rk.order, order_b))
        out[name]["ranking_agreement"] = 1.0 - inv / total
        out[name]["concordance_s"] = t
        out[name]["top100_equal"] = bool(np.array_equal(order_b[:100], rk.order[:100]))
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
