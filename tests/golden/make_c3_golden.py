"""Golden results for C3 (R-MAT scale 27, edge factor 16, seed 42, undirected,
TopK(100, 1e-6)) -- the north-star configuration -- computed by the CPU
oracle.  TEST INFRASTRUCTURE; run once in the build container:

    python tests/golden/make_c3_golden.py      # ~15-25 min, ~40 GB RAM

Writes tests/golden/c3.json.  Nothing at GPU-test time recomputes this.

Why the oracle and not the reference itself: the reference's own CSR for
this graph (scipy, int64 indices + fp64 data) needs ~67 GB
of host memory, more than this container has.  The oracle is the reference
restated (oracle/katz_oracle.py, every function citing engine.py lines) and
is pinned bit for bit to the reference's own digests at C1, s20 and C2
(tests/test_oracle.py), so its C3 digests are the
reference's up to that pinning.  Its generator is the low-memory variant of
the pinned R-MAT sampler (same unique key set; checked equal at s16 in
tests/test_oracle.py).

Recorded: n, nnz, deg_max, alpha, gamma, the iteration count r, the
per-check active-set sizes, the separated fraction and exact pair count,
top-10, the k-boundary certification margin, sha256[:16] digests of the
full order (int64), of lower and upper (fp64, every row one sequential sum
= scipy csr_matvec), of the top-100, and the exact bounds of a fixed node
sample (the top 1000 plus 4096 seeded random ids) for 1e-12 checks of the
default (segmented) device layout.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import katz_oracle as O  # noqa: E402


def h16(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def main(scale: int = 27, out_name: str = "c3.json") -> None:
    t0 = time.time()
    n = 1 << scale
    threads = os.cpu_count() or 1
    g = O.rmat_graph_lowmem(n, edge_factor=16, seed=42, threads=threads)
    print(f"graph: n={n} nnz={g.nnz} deg_max={g.max_out_degree()} "
          f"({time.time() - t0:.0f}s)", flush=True)
    crit = O.Crit(O.TOPK, epsilon=1e-6, k=100)
    st = O.OracleState(g, crit, undirected=True, threads=threads)
    active_sizes = []
    while True:
        t1 = time.time()
        O.iterate_once(st, g)
        done = O.check_converged(st)
        active_sizes.append(int(st.active.size))
        print(f"r={st.r} active={st.active.size} ({time.time() - t1:.0f}s)",
              flush=True)
        if done:
            break
        assert st.r < st.max_iterations
    margin_hi = float(st.lower[st.active[99]])
    res = O.ranking_result(st)
    order = res.order
    second = order[100]
    rng = np.random.default_rng(2027)
    sample = np.unique(np.concatenate([order[:1000],
                                       rng.integers(0, n, size=4096)]))
    out = dict(
        workload="rmat-s%d-ef16-topk100" % scale, scale=scale, n=n, nnz=g.nnz,
        deg_max=g.max_out_degree(), alpha=st.alpha.hex(), gamma=st.gamma.hex(),
        r=res.iterations_used, active_sizes=active_sizes,
        sepfrac=res.separated_fraction, separated_pairs=res.separated_pairs,
        top10=res.top(10),
        k_margin=[margin_hi, float(st.upper[second])],
        order=h16(order.astype(np.int64)), lower=h16(res.lower),
        upper=h16(res.upper),
        top100=h16(np.asarray(res.top(100), dtype=np.int64)),
        sample_ids=sample.tolist(),
        sample_lower=[float(x).hex() for x in res.lower[sample]],
        sample_upper=[float(x).hex() for x in res.upper[sample]],
        generator="oracle.rmat_graph_lowmem (pinned sampler)",
        seconds=round(time.time() - t0, 1),
    )
    with open(os.path.join(HERE, out_name), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: v for k, v in out.items() if not k.startswith("sample")}),
          flush=True)


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 27,
         sys.argv[2] if len(sys.argv) > 2 else "c3.json")
