"""Generate golden vectors by running the *reference* katzbounds package.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

Writes tests/golden/small_cases.npz, dynamic_cases.npz and digests.json.
The reference is imported read-only from /root/reference/pkg/src with
bytecode writing disabled.  Nothing at test time reads /root/reference.
"""
from __future__ import annotations

import hashlib
import json
import os
import random
import sys

sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, "/root/reference/pkg/tests")

import numpy as np  # noqa: E402

import katzbounds as K  # noqa: E402
import builders  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def h16(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def edges_of(g):
    return np.array(sorted(g.arcs()), dtype=np.int64).reshape(-1, 2)


def small_graphs():
    """(name, graph, undirected) drawn from the reference test builders."""
    out = [
        ("star7", builders.star(7), True),
        ("path9", builders.path(9), True),
        ("cycle5", builders.cycle(5), True),
        ("k6", builders.complete(6), True),
        ("grid6x7", builders.grid(6, 7), True),
        ("grid16x16", builders.grid(16, 16), True),
        ("dpath3", K.Graph.from_edges(3, [(0, 1), (1, 2)]), False),
        ("edgeless4", K.Graph.from_edges(4, []), False),
        ("single1", K.Graph.from_edges(1, []), False),
    ]
    for seed in range(6):
        out.append((f"er{seed}", builders.er_graph(60 + 10 * seed, 0.08, seed=seed), True))
    for seed in range(3):
        out.append((f"der{seed}", builders.er_graph(40, 0.08, seed=50 + seed,
                                                   undirected=False), False))
    # isolated nodes mixed in (relabeling must keep them last-and-zero)
    out.append(("sparse200", builders.er_graph(200, 0.006, seed=9), True))
    return out


def criteria(n):
    cs = [("ranking", K.Criterion.ranking(1e-8)),
          ("score", K.Criterion.score(1e-9))]
    if n >= 3:
        cs.append(("topk", K.Criterion.top_k(min(3, n), 1e-7)))
    if n >= 2:
        cs.append(("pair", K.Criterion.pair(0, n - 1, 1e-6)))
    return cs


def make_small():
    arrays = {}
    index = []
    for name, g, und in small_graphs():
        n = g.node_count
        arrays[f"{name}/edges"] = edges_of(g)
        for cname, crit in criteria(n):
            key = f"{name}/{cname}"
            st = K.init(g, crit, undirected=und)
            try:
                res = K.run(st, g)
            except K.ConvergenceError:
                continue
            arrays[f"{key}/order"] = np.asarray(res.order, dtype=np.int64)
            arrays[f"{key}/lower"] = np.asarray(res.lower)
            arrays[f"{key}/upper"] = np.asarray(res.upper)
            arrays[f"{key}/katz"] = np.asarray(st.katz)
            arrays[f"{key}/levels"] = np.stack(st.levels)
            arrays[f"{key}/active"] = np.sort(np.asarray(st.active, dtype=np.int64))
            index.append(dict(key=key, graph=name, n=n, undirected=und,
                              kind=crit.kind, epsilon=crit.epsilon, k=crit.k,
                              u=crit.u, v=crit.v, alpha=st.alpha,
                              gamma=st.gamma, r=res.iterations_used,
                              sepfrac=res.separated_fraction,
                              max_iterations=st.max_iterations))
    np.savez_compressed(os.path.join(HERE, "small_cases.npz"), **arrays)
    return index


def make_dynamic():
    """Batches applied with the reference update_batch; record the state."""
    arrays = {}
    index = []
    cases = [
        ("er_und", builders.er_graph(35, 0.1, seed=2), True, K.Criterion.ranking(1e-7), 0.02, 1.0),
        ("er_und_theta0", builders.er_graph(30, 0.1, seed=5), True, K.Criterion.score(1e-9), 0.05, 0.0),
        ("grid_topk", builders.grid(8, 8), True, K.Criterion.top_k(4, 1e-8), None, 0.5),
        ("er_dir", builders.er_graph(40, 0.08, seed=13, undirected=False), False, K.Criterion.score(1e-9), 0.05, 1.0),
    ]
    for name, g, und, crit, alpha, theta in cases:
        rng = random.Random(hash(name) & 0xffff)
        arrays[f"{name}/edges0"] = edges_of(g)
        st = K.init(g, crit, alpha=alpha, undirected=und)
        K.run(st, g)
        steps = []
        for b in range(4):
            batch = builders.random_batch(g, rng, max_ops=4, undirected=und)
            try:
                K.update_batch(st, g, batch, theta=theta)
            except K.ParameterError:
                continue
            p = f"{name}/b{len(steps)}"
            arrays[p + "/ins"] = np.array(batch.insertions, dtype=np.int64).reshape(-1, 2)
            arrays[p + "/del"] = np.array(batch.deletions, dtype=np.int64).reshape(-1, 2)
            arrays[p + "/lower"] = st.lower.copy()
            arrays[p + "/upper"] = st.upper.copy()
            arrays[p + "/katz"] = st.katz.copy()
            arrays[p + "/levels"] = np.stack(st.levels)
            arrays[p + "/active"] = np.sort(np.asarray(st.active, dtype=np.int64))
            s = st.last_update_stats
            steps.append(dict(r=st.r, seeds=s.seeds, visited=s.visited,
                              level_sizes=list(s.level_sizes),
                              reactivated=s.reactivated,
                              aborted_level=s.aborted_level,
                              resumed_iterations=s.resumed_iterations,
                              gamma=st.gamma))
        index.append(dict(name=name, n=g.node_count, undirected=und,
                          kind=crit.kind, epsilon=crit.epsilon, k=crit.k,
                          alpha=st.alpha, theta=theta, steps=steps))
    np.savez_compressed(os.path.join(HERE, "dynamic_cases.npz"), **arrays)
    return index


def run_digest(g, crit, und=True):
    st = K.init(g, crit, undirected=und)
    res = K.run(st, g)
    return dict(r=res.iterations_used, sepfrac=res.separated_fraction,
                alpha=st.alpha, gamma=st.gamma, max_iterations=st.max_iterations,
                top10=res.top(10),
                top100=[int(x) for x in res.order[:100]],
                order=h16(np.asarray(res.order, dtype=np.int64)),
                lower=h16(res.lower), upper=h16(res.upper),
                top100_digest=h16(np.asarray(res.order[:100], dtype=np.int64)),
                lower_top100=[float(res.lower[v]) for v in res.order[:100]],
                upper_top100=[float(res.upper[v]) for v in res.order[:100]],
                active=int(st.active.size))


class _CSRShim:
    """Duck-typed CSR graph for the reference engine."""

    def __init__(self, n, edges):
        from scipy import sparse
        src = np.concatenate([edges[:, 0], edges[:, 1]])
        dst = np.concatenate([edges[:, 1], edges[:, 0]])
        key = np.unique(src * n + dst)
        rows, cols = key // n, key % n
        indptr = np.zeros(n + 1, dtype=np.int64)
        np.add.at(indptr, rows + 1, 1)
        np.cumsum(indptr, out=indptr)
        self.node_count = n
        self.version = 1
        self._deg = np.diff(indptr)
        self._csr = sparse.csr_matrix((np.ones(key.size), cols.astype(np.int32), indptr),
                                      shape=(n, n))
        self.indptr, self.indices = indptr, cols

    def max_out_degree(self):
        return int(self._deg.max())

    def is_symmetric(self):
        return True

    def out_csr(self):
        return self._csr


def make_digests():
    d = {}
    # PCG64 raw stream, numpy's bit generator, seed 42 (generate.py:68)
    raw = np.random.default_rng(42).bit_generator.random_raw(64)
    d["pcg64_seed42_raw64"] = [int(x) for x in raw]
    st = np.random.default_rng(42).bit_generator.state["state"]
    d["pcg64_seed42_state"] = [str(st["state"]), str(st["inc"])]
    for ef in (8, 16):
        e = np.array(K.generate("rmat", 65536, seed=42, edge_factor=ef), dtype=np.int64)
        d[f"rmat_s16_ef{ef}_edges"] = dict(count=int(e.shape[0]),
                                            packed=h16(e[:, 0] * 65536 + e[:, 1]))
        shim = _CSRShim(65536, e)
        d[f"rmat_s16_ef{ef}_csr"] = dict(nnz=int(shim.indptr[-1]),
                                          dmax=shim.max_out_degree(),
                                          indptr=h16(shim.indptr),
                                          indices=h16(shim.indices.astype(np.int32)))
        if ef == 16:
            d["C1_topk100"] = run_digest(shim, K.Criterion.top_k(100, 1e-6))
        else:
            d["fixture_ranking1e-6"] = run_digest(shim, K.Criterion.ranking(1e-6))
            d["fixture_eps_sweep"] = []
            for eps in [10.0 ** -i for i in range(1, 13)]:
                st2 = K.init(shim, K.Criterion.ranking(eps), undirected=True)
                res2 = K.run(st2, shim)
                d["fixture_eps_sweep"].append([eps, res2.iterations_used,
                                               res2.separated_fraction])
    # grid 256^2 ranking(1e-9): exact ties decided by rounding
    ge = np.array(K.generate("grid", 256 * 256), dtype=np.int64)
    d["grid256_ranking1e-9"] = run_digest(_CSRShim(256 * 256, ge), K.Criterion.ranking(1e-9))
    # rmat s12 with topk and score on the real Graph type
    e12 = K.generate("rmat", 4096, seed=3, edge_factor=16)
    g12 = K.Graph.from_edges(4096, e12, undirected=True)
    d["rmat_s12_seed3_topk50"] = run_digest(g12, K.Criterion.top_k(50, 1e-9))
    return d


def main():
    idx_small = make_small()
    idx_dyn = make_dynamic()
    dig = make_digests()
    with open(os.path.join(HERE, "digests.json"), "w") as fh:
        json.dump(dict(small=idx_small, dynamic=idx_dyn, digests=dig), fh,
                  indent=1)
    print("small cases", len(idx_small), "dynamic", len(idx_dyn))


if __name__ == "__main__":
    main()
