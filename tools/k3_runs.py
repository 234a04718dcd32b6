"""K3 sort experiment: how the C2 bounds cluster under a 32-bit leading-key
sort (keys offset by their minimum) -- run lengths and out-of-order runs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1807_03847_b200 as P  # noqa: E402
from paper_1807_03847_b200 import generators as G  # noqa: E402

SCALE = int(os.environ.get("SCALE", "24"))
for name, g, crit in (("c%d" % (2 if SCALE == 24 else 3), lambda: G.rmat_graph(1 << SCALE, edge_factor=16, seed=42),
                       P.Criterion.top_k(100, 1e-6)),
                      ("c4", lambda: G.grid_graph(1 << 24), P.Criterion.ranking(1e-9))):
    g = g()
    st = P.init(g, crit, undirected=True, max_iterations=200)
    P.run(st, g)
    lo = np.asarray(st.lower)
    pos = np.nonzero(lo > 0)[0]
    key = ~lo[pos].view(np.uint64)
    mn, mx = key.min(), key.max()
    d = int(mx - mn)
    for hb in tuple(int(x) for x in os.environ.get('HBITS', '32,28,24').split(',')):
        s = max(0, d.bit_length() - hb)
        hi = ((key - mn) >> np.uint64(s)).astype(np.uint64)
        o = np.argsort(hi, kind="stable")
        hs, ks = hi[o], key[o]
        start = np.ones(hs.size, bool)
        start[1:] = hs[1:] != hs[:-1]
        rid = np.cumsum(start) - 1
        viol = np.zeros(hs.size, bool)
        viol[1:] = (hs[1:] == hs[:-1]) & (ks[:-1] > ks[1:])
        runs = np.bincount(rid)
        bad = np.unique(rid[viol])
        print(f"{name} hbits={hb} shift={s} npos={pos.size} runs={runs.size} "
              f"maxrun={runs.max()} runs>1={np.sum(runs > 1)} bad_runs={bad.size} "
              f"bad_elems={runs[bad].sum() if bad.size else 0} "
              f"max_bad={runs[bad].max() if bad.size else 0}", flush=True)
    del st, g
