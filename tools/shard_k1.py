"""K1 time of one rank's shard at P ranks, on one GPU (no collectives: the
omega vector is left as iterated locally, which does not change the work).
Projects the per-rank SpMV cost of the sharded path and the effect of the
per-block hot set (kb_tune k1.shard_hot).

  python tools/shard_k1.py [P ...]
"""
from __future__ import annotations

import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1807_03847_b200 as P  # noqa: E402
from paper_1807_03847_b200 import _lib  # noqa: E402
from paper_1807_03847_b200 import distributed as D  # noqa: E402
from paper_1807_03847_b200 import generators as G  # noqa: E402


def main():
    worlds = [int(x) for x in sys.argv[1:]] or [1, 2, 4, 8]
    L = _lib.lib()
    g = G.rmat_graph(1 << int(os.environ.get("SCALE", "24")), edge_factor=16, seed=42)
    ip, ix = g.csr_arrays()
    g.device_graph.close()
    crit = P.Criterion.top_k(100, 1e-6)
    for world in worlds:
        plan = D.ShardPlan(ip, world)
        d = plan.max_degree
        alpha = 1.0 / (1.0 + d)
        gamma = P.tail_gamma(alpha, d)
        sh = D.CudaShard(plan, 0, ip, ix, device=0, alpha=alpha, gamma=gamma, crit=crit,
                         undirected=True, max_iterations=200,
                         split_threshold=int(os.environ.get("SPLIT", "0")))
        for hot in (1, 0):
            _lib.check(L.kb_tune(b"k1.shard_hot", hot))
            _lib.check(L.kb_tune(b"k1.depth", int(os.environ.get("DEPTH", "1"))))
            if "HEAVY" in os.environ:
                _lib.check(L.kb_tune(b"k1.heavy_warp", int(os.environ["HEAVY"])))
            sh.reset(alpha=alpha, gamma=gamma, crit=crit, undirected=True, max_iterations=200)
            for _ in range(7):
                sh.iterate()
            info = _lib.StateInfo()
            _lib.check(L.kb_state_info_get(sh.s, ctypes.byref(info)))
            per = info.spmv_ms / max(1, info.spmv_launches)
            print(f"P={world} rank0 shard: K1 {per:.3f} ms/iter over {info.spmv_launches} "
                  f"launches (shard_hot={hot}); single-GPU K1 / P = see bench", flush=True)
        _lib.check(L.kb_tune(b"k1.shard_hot", 1))
        sh.close()


if __name__ == "__main__":
    main()
