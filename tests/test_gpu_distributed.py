"""The CUDA shard backend on one B200.

Two ranks whose kernels wait on each other must not share one GPU, so the
P=2 protocol is driven here in lockstep inside one process: both shards live
on cuda:0 and the all-gather is a device copy between their omega blocks.
The result must equal the single-GPU engine bit for bit (same per-row sums,
same segmentation) and the oracle's certified order."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import katz_oracle as O

pytestmark = pytest.mark.gpu

P = pytest.importorskip("paper_1807_03847_b200")
torch = pytest.importorskip("torch")
from paper_1807_03847_b200 import distributed as D  # noqa: E402


def _lockstep(g0, crit, world, protocol="device", split=0):
    plan = D.ShardPlan(g0.indptr, world)
    d = plan.max_degree
    alpha = 1.0 / (1.0 + d)
    gamma = P.tail_gamma(alpha, d)
    cap = P.default_iteration_cap(alpha, d, crit.epsilon)
    shards = [D.CudaShard(plan, rk, g0.indptr, g0.indices, device=0, alpha=alpha,
                          gamma=gamma, crit=crit, undirected=True, max_iterations=cap,
                          split_threshold=split)
              for rk in range(world)]
    n_per = plan.n_per
    r = 0
    while True:
        for s in shards:
            s.iterate()
        torch.cuda.synchronize()
        r += 1
        lv = [s.level_tensor() for s in shards]
        for rk in range(world):               # all-gather by device copies
            blk = lv[rk][rk * n_per:(rk + 1) * n_per].clone()
            for other in range(world):
                if other != rk:
                    lv[other][rk * n_per:(rk + 1) * n_per].copy_(blk)
        torch.cuda.synchronize()
        if crit.kind == "score":
            done = max(s.local_gap() for s in shards) < crit.epsilon
        elif protocol == "device":
            k = int(crit.k)
            blks = [s.new_buffer(1 + 3 * k) for s in shards]
            words = [s.new_buffer(3) for s in shards]
            torch.cuda.synchronize()
            for s, b in zip(shards, blks):
                s.propose(k, b)
            torch.cuda.synchronize()
            allb = torch.cat(blks)
            torch.cuda.synchronize()
            for s, w in zip(shards, words):
                s.cut(allb, world, k, w)
            torch.cuda.synchronize()
            ws = [w.tolist() for w in words]
            assert len({w[2] for w in ws}) == 1
            for s, w in zip(shards, ws):
                s.commit(w[1])
            done = sum(w[0] for w in ws) <= k and bool(ws[0][2])
        else:
            k = int(crit.k)
            props = [s.local_topk(k) for s in shards]
            keys = np.concatenate([p[0] for p in props])
            labs = np.concatenate([p[1] for p in props])
            ups = np.concatenate([p[2] for p in props])
            cuts = [s.select_global(keys, labs, ups, k, crit.epsilon) for s in shards]
            assert len(set(cuts)) == 1           # every rank takes the same cut
            kstar, istar, ok = cuts[0]
            m = sum(s.apply_cut(kstar, istar) for s in shards)
            done = m <= k and ok
        if done:
            break
        assert r < 64
    lo = [s.bounds_tensors() for s in shards]
    node = plan.node_of_exch
    valid = node >= 0
    lower = np.empty(plan.n)
    upper = np.empty(plan.n)
    for rk in range(world):
        a, b = plan.block(rk)
        sel = valid[a:b]
        lower[node[a:b][sel]] = lo[rk][0][a:b].cpu().numpy()[sel]
        upper[node[a:b][sel]] = lo[rk][1][a:b].cpu().numpy()[sel]
    order, pairs = shards[0].rank_bounds(lower, upper)
    # the device result path: gather every block into shard 0's bounds
    lo0, up0 = lo[0]
    for rk in range(1, world):
        a, b = plan.block(rk)
        lo0[a:b].copy_(lo[rk][0][a:b])
        up0[a:b].copy_(lo[rk][1][a:b])
    torch.cuda.synchronize()
    o2, l2, u2, p2 = shards[0].rank_gathered()
    np.testing.assert_array_equal(o2, order)
    np.testing.assert_array_equal(l2, lower)
    np.testing.assert_array_equal(u2, upper)
    assert p2 == pairs
    assert shards[0].rank_gathered(host=False)[3] == pairs
    for s in shards:
        s.close()
    return r, order, lower, upper, pairs


@pytest.mark.parametrize("world,protocol", [(1, "device"), (2, "device"), (3, "device"),
                                            (2, "host")])
def test_cuda_shards_equal_single_gpu(world, protocol):
    g0 = O.rmat_graph(1 << 14, edge_factor=16, seed=42)
    crit = P.Criterion.top_k(100, 1e-6)
    r, order, lower, upper, pairs = _lockstep(g0, crit, world, protocol)
    g = P.Graph.from_csr(g0.node_count, g0.indptr, g0.indices)
    res = P.run(P.init(g, crit, undirected=True), g)
    assert r == res.iterations_used
    np.testing.assert_array_equal(order, res.order)
    np.testing.assert_array_equal(lower, res.lower)
    np.testing.assert_array_equal(upper, res.upper)
    n = g0.node_count
    assert pairs / (n * (n - 1) // 2) == res.separated_fraction
    ores = O.run(O.OracleState(g0, O.Crit("topk", 1e-6, k=100)), g0)
    assert ores.top(100) == [int(v) for v in order[:100]]


def test_cuda_shards_score_criterion():
    g0 = O.rmat_graph(1 << 12, edge_factor=16, seed=3)
    crit = P.Criterion.score(1e-7)
    r, order, lower, upper, _ = _lockstep(g0, crit, 2)
    ost = O.OracleState(g0, O.Crit("score", 1e-7))
    ores = O.run(ost, g0)
    assert r == ores.iterations_used
    np.testing.assert_allclose(lower, ores.lower, rtol=1e-12, atol=0)
    np.testing.assert_array_equal(order, ores.order)


def test_cuda_shards_fast_split_within_tolerance():
    """The bench's finer row segmentation (fast_split) changes only the
    rounding of long rows: same iterations and order, bounds within 1e-12."""
    g0 = O.rmat_graph(1 << 14, edge_factor=16, seed=42)
    crit = P.Criterion.top_k(100, 1e-6)
    r, order, lower, upper, pairs = _lockstep(g0, crit, 4, split=D.fast_split(8) // 2)
    g = P.Graph.from_csr(g0.node_count, g0.indptr, g0.indices)
    res = P.run(P.init(g, crit, undirected=True), g)
    assert r == res.iterations_used
    np.testing.assert_array_equal(order[:100], res.order[:100])
    np.testing.assert_allclose(lower, res.lower, rtol=1e-12, atol=0)
    np.testing.assert_allclose(upper, res.upper, rtol=1e-12, atol=0)
