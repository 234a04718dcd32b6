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


def _lockstep(g0, crit, world, protocol="device", split=0, fused=False, build="host"):
    """build="device": every shard is cut out of one device graph on the GPU
    (kb_graph_create_shard) instead of from the plan's host CSR slice."""
    plan = D.ShardPlan(g0.indptr, world)
    d = plan.max_degree
    alpha = 1.0 / (1.0 + d)
    gamma = P.tail_gamma(alpha, d)
    cap = P.default_iteration_cap(alpha, d, crit.epsilon)
    full = P.DeviceGraph(g0.indptr, g0.indices, device=0) if build == "device" else None
    shards = [D.CudaShard(plan, rk, g0.indptr, g0.indices, device=0, alpha=alpha,
                          gamma=gamma, crit=crit, undirected=True, max_iterations=cap,
                          split_threshold=split, fused=fused, full=full,
                          host_build=build == "gather")
              for rk in range(world)]
    if full is not None:
        full.close()
    if fused:                                 # peers are buffers in this process
        exports = [s.exchange_export() for s in shards]
        for s in shards:
            s.exchange_connect(exports, same_process=True)
    n_per = plan.n_per
    r = 0
    while True:
        for s in shards:
            s.iterate()
        torch.cuda.synchronize()
        r += 1
        if not fused:
            lv = [s.level_tensor() for s in shards]
            for rk in range(world):           # all-gather by device copies
                blk = lv[rk][rk * n_per:(rk + 1) * n_per].clone()
                for other in range(world):
                    if other != rk:
                        lv[other][rk * n_per:(rk + 1) * n_per].copy_(blk)
        torch.cuda.synchronize()
        if crit.kind == "score":
            done = max(s.local_gap() for s in shards) < crit.epsilon
        elif crit.kind == "ranking":
            bt = [s.bounds_tensors() for s in shards]
            for rk in range(world):           # gather the bound blocks
                a, b = rk * n_per, (rk + 1) * n_per
                for other in range(world):
                    if other != rk:
                        bt[other][0][a:b].copy_(bt[rk][0][a:b])
                        bt[other][1][a:b].copy_(bt[rk][1][a:b])
            torch.cuda.synchronize()
            verdicts = {s.check_full() for s in shards}
            assert len(verdicts) == 1             # every rank decides the same
            done = verdicts.pop()
        elif crit.kind == "pair":
            vals = np.sum([s.pair_values(crit.u, crit.v) for s in shards], axis=0)
            lu, uu, lv, uv = (float(x) for x in vals)
            lw, ux = (lu, uv) if (lu, -crit.u) >= (lv, -crit.v) else (lv, uu)
            done = lw > ux - crit.epsilon
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
        assert r < 400
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


@pytest.mark.parametrize("world,protocol,fused,build",
                         [(1, "device", False, "host"), (2, "device", False, "host"),
                          (3, "device", False, "host"), (2, "host", False, "host"),
                          (2, "device", True, "host"), (3, "host", True, "host"),
                          (1, "device", False, "device"), (3, "device", False, "device"),
                          (4, "device", True, "device"), (2, "device", False, "gather"),
                          (5, "device", True, "gather")])
def test_cuda_shards_equal_single_gpu(world, protocol, fused, build):
    """fused: K1 stores omega straight into the other shards' level buffers
    (the NVLink exchange), no all-gather.  build="device": shards cut out of
    a device graph on the GPU (kb_graph_create_shard); build="gather": from the
    host CSR, only indptr and the rank's rows uploaded
    (kb_graph_create_shard_host)."""
    g0 = O.rmat_graph(1 << 14, edge_factor=16, seed=42)
    crit = P.Criterion.top_k(100, 1e-6)
    r, order, lower, upper, pairs = _lockstep(g0, crit, world, protocol, fused=fused,
                                              build=build)
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


@pytest.mark.parametrize("fused", [False, True])
def test_cuda_shards_score_criterion(fused):
    g0 = O.rmat_graph(1 << 12, edge_factor=16, seed=3)
    crit = P.Criterion.score(1e-7)
    r, order, lower, upper, _ = _lockstep(g0, crit, 2, fused=fused)
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


def _ipc_rank(rank, world, port, out_dir):
    """One process of the two-process fused-exchange test (both on cuda:0;
    host barriers only, so neither rank's kernels wait on the other)."""
    import os
    import pickle

    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g0 = O.rmat_graph(1 << 12, edge_factor=16, seed=7)
    crit = P.Criterion.top_k(50, 1e-6)
    plan = D.ShardPlan(g0.indptr, world)
    d = plan.max_degree
    alpha = 1.0 / (1.0 + d)
    sh = D.CudaShard(plan, rank, g0.indptr, g0.indices, device=0, alpha=alpha,
                     gamma=P.tail_gamma(alpha, d), crit=crit, undirected=True,
                     max_iterations=100, fused=True)
    exports = [None] * world
    dist.all_gather_object(exports, sh.exchange_export())
    sh.exchange_connect(exports)              # CUDA IPC handles of the other process
    r = 0
    while True:
        sh.iterate()
        sh.sync()
        dist.barrier()                        # every rank's stores have landed
        r += 1
        props = [None] * world
        dist.all_gather_object(props, sh.local_topk(50))
        keys = np.concatenate([p[0] for p in props])
        labs = np.concatenate([p[1] for p in props])
        ups = np.concatenate([p[2] for p in props])
        kstar, istar, ok = sh.select_global(keys, labs, ups, 50, 1e-6)
        m = [None] * world
        dist.all_gather_object(m, sh.apply_cut(kstar, istar))
        if sum(m) <= 50 and ok:
            break
    lo, up = sh.bounds_tensors()
    a, b = plan.block(rank)
    with open(os.path.join(out_dir, f"rank{rank}.pkl"), "wb") as fh:
        pickle.dump((r, a, b, lo[a:b].cpu().numpy(), up[a:b].cpu().numpy()), fh)
    sh.close()
    dist.barrier()
    dist.destroy_process_group()


def test_fused_exchange_two_processes_ipc(tmp_path):
    """Two processes exchange omega through CUDA IPC mappings of each other's
    level buffers; the certified bounds equal the single-GPU engine's."""
    import pickle
    import socket

    import torch.multiprocessing as mp
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    mp.start_processes(_ipc_rank, args=(2, port, str(tmp_path)), nprocs=2, join=True,
                       start_method="spawn")
    g0 = O.rmat_graph(1 << 12, edge_factor=16, seed=7)
    plan = D.ShardPlan(g0.indptr, 2)
    lower = np.empty(plan.n)
    upper = np.empty(plan.n)
    node = plan.node_of_exch
    rs = set()
    for rank in range(2):
        with open(tmp_path / f"rank{rank}.pkl", "rb") as fh:
            r, a, b, lo, up = pickle.load(fh)
        rs.add(r)
        sel = node[a:b] >= 0
        lower[node[a:b][sel]] = lo[sel]
        upper[node[a:b][sel]] = up[sel]
    g = P.Graph.from_csr(g0.node_count, g0.indptr, g0.indices)
    res = P.run(P.init(g, P.Criterion.top_k(50, 1e-6), undirected=True), g)
    assert rs == {res.iterations_used}
    np.testing.assert_array_equal(lower, res.lower)
    np.testing.assert_array_equal(upper, res.upper)


def test_sharded_run_one_rank_nccl_speculative():
    """sharded_run end to end on one rank over NCCL: the per-check host read
    overlaps a speculative K1 of the next level (rolled back at
    convergence); the result equals the single-GPU engine's bit for bit."""
    import socket

    import torch.distributed as dist
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0,
                            world_size=1, device_id=torch.device("cuda", 0))
    try:
        g0 = O.rmat_graph(1 << 14, edge_factor=16, seed=42)
        crit = P.Criterion.top_k(100, 1e-6)
        res = D.sharded_run(g0.indptr, g0.indices, crit, device=0, undirected=True)
        # engine.init's guards (engine.py:257-283) hold for sharded runs too
        # drop row 0's last arc: its reversal stays, so the set is asymmetric
        cut = int(g0.indptr[1]) - 1
        ix_bad = np.delete(g0.indices, cut)
        ip_bad = g0.indptr.copy()
        ip_bad[1:] -= 1
        with pytest.raises(P.ParameterError, match="symmetric"):
            D.sharded_run(ip_bad, ix_bad, crit, device=0, undirected=True)
        with pytest.raises(P.ParameterError, match="exceeds"):
            D.sharded_run(g0.indptr, g0.indices, P.Criterion.top_k(g0.node_count + 1),
                          device=0, undirected=True)
        with pytest.raises(P.ParameterError, match="max_iterations"):
            D.sharded_run(g0.indptr, g0.indices, crit, device=0, undirected=True,
                          max_iterations=0)
        # the host-gather shard's distributed symmetry check through NCCL's
        # all-to-all (the path sharded_run takes at more than one rank)
        plan = D.DevicePlan(g0.node_count, 1, int(np.diff(g0.indptr).max()))
        for ip, ix, sym in ((g0.indptr, g0.indices, True), (ip_bad, ix_bad, False)):
            sh = D.CudaShard(plan, 0, ip, ix, device=0, alpha=1e-4, gamma=1.0, crit=crit,
                             undirected=True, max_iterations=10, host_build=True)
            assert D.shards_symmetric(sh, dist, 1) == sym
            sh.close()
    finally:
        dist.destroy_process_group()
    g = P.Graph.from_csr(g0.node_count, g0.indptr, g0.indices)
    ref = P.run(P.init(g, crit, undirected=True), g)
    assert res.iterations_used == ref.iterations_used
    np.testing.assert_array_equal(res.order, ref.order)
    np.testing.assert_array_equal(res.lower, ref.lower)
    np.testing.assert_array_equal(res.upper, ref.upper)
    assert res.separated_fraction == ref.separated_fraction


@pytest.mark.parametrize("kind,world,fused", [("ranking", 2, False), ("ranking", 3, True),
                                              ("pair", 2, False), ("pair", 3, True)])
def test_cuda_shards_ranking_and_pair_equal_single_gpu(kind, world, fused):
    """Sharded RANKING (every rank certifies the gathered bounds with the
    O(n) certificates) and PAIR (the two nodes' bounds all-reduced from their
    owners) reproduce the single-GPU run bit for bit (engine.py:346-378)."""
    if kind == "ranking":
        g0 = O.grid_graph(48 * 48)
        crit = P.Criterion.ranking(1e-9)
    else:
        g0 = O.rmat_graph(1 << 14, edge_factor=16, seed=42)
        crit = P.Criterion.pair(16, 256, 1e-9)
    r, order, lower, upper, pairs = _lockstep(g0, crit, world, fused=fused, build="device")
    g = P.Graph.from_csr(g0.node_count, g0.indptr, g0.indices)
    res = P.run(P.init(g, crit, undirected=True), g)
    assert r == res.iterations_used
    np.testing.assert_array_equal(order, res.order)
    np.testing.assert_array_equal(lower, res.lower)
    np.testing.assert_array_equal(upper, res.upper)


@pytest.mark.parametrize("world,fused", [(3, True), (4, False)])
def test_cuda_shards_s20_match_reference_digests(world, fused):
    """R-MAT s20 (31.4M arcs) on 3-4 lockstep shards with sequential rows:
    r, order, bounds and separated fraction bit-identical to the reference's
    own run (SURVEY.md §8(c) digests)."""
    import hashlib

    def h16(a):
        return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]

    g0 = O.rmat_graph(1 << 20, edge_factor=16, seed=42)
    crit = P.Criterion.top_k(100, 1e-6)
    r, order, lower, upper, pairs = _lockstep(g0, crit, world, split=1 << 30, fused=fused)
    n = g0.node_count
    assert r == 7
    assert [int(v) for v in order[:10]] == [0, 2048, 32768, 131072, 4096, 4, 256, 524288,
                                            1024, 32]
    assert pairs / (n * (n - 1) // 2) == 0.8525977645781982
    assert h16(np.asarray(order, dtype=np.int64)) == "85ea50d05c5dfd0e"
    assert h16(lower) == "f13ddf321fb10751"
    assert h16(upper) == "9db3105f69a9e233"


@pytest.mark.parametrize("world", [1, 3, 8])
def test_device_shard_csr_equals_host_plan(world):
    """kb_graph_create_shard builds exactly the CSR the host ShardPlan
    describes (exchange ids, owned rows only, original arc order), also from
    a mutated device graph (degree order re-sorted on the device)."""
    import ctypes

    from paper_1807_03847_b200 import _lib
    g0 = O.rmat_graph(1 << 13, edge_factor=16, seed=9)
    L = _lib.lib()
    for mutated in (False, True):
        ip, ix = g0.indptr, g0.indices
        dg = P.DeviceGraph(ip, ix, device=0)
        if mutated:        # drop two arcs (u, v), (v, u) on the device
            u, v = 0, int(ix[ip[0]])
            dels = np.array([[u, v], [v, u]], dtype=np.int64)
            _lib.check(L.kb_graph_apply_batch(dg.handle, None, 0, _lib.ptr(dels), 2))
            keep = np.ones(ix.size, dtype=bool)
            keep[ip[0]] = False
            keep[ip[v] + np.searchsorted(ix[ip[v]:ip[v + 1]], u)] = False
            ix = ix[keep]
            ip = np.concatenate([[0], np.cumsum(np.diff(g0.indptr) - np.bincount(
                [u, v], minlength=g0.node_count))]).astype(np.int64)
        plan = D.ShardPlan(ip, world)
        for rank in range(world):
            h, n_per, owned = ctypes.c_void_p(), ctypes.c_int64(), ctypes.c_int64()
            _lib.check(L.kb_graph_create_shard(dg.handle, world, rank, 0, -1, ctypes.byref(h),
                                               ctypes.byref(n_per), ctypes.byref(owned)))
            assert (n_per.value, owned.value) == (plan.n_per, plan.owned(rank))
            N = world * plan.n_per
            info = _lib.GraphInfo()
            _lib.check(L.kb_graph_info_get(h, ctypes.byref(info)))
            dip = np.empty(N + 1, dtype=np.int64)
            dix = np.empty(int(info.nnz), dtype=np.int32)
            _lib.check(L.kb_graph_get_csr(h, _lib.ptr(dip), _lib.ptr(dix)))
            hip, hix = plan.local_csr(ip, ix, rank)
            np.testing.assert_array_equal(dip, hip)
            np.testing.assert_array_equal(dix, hix)
            L.kb_graph_destroy(h)
        dg.close()


def _exchange_symmetry(shards):
    """shards_symmetric's all-to-all, by hand between lockstep shards."""
    parts = [s.symmetry_keys() for s in shards]
    oks = []
    for q, s in enumerate(shards):
        recv = []
        for keys, counts in parts:
            a = sum(counts[:q])
            recv.append(keys[a:a + counts[q]])
        oks.append(s.symmetry_verify(torch.cat(recv)))
    return oks


@pytest.mark.parametrize("world", [1, 2, 5])
def test_host_gather_shards_decide_symmetry_exactly(world):
    """kb_graph_create_shard_host + the distributed symmetry check: every
    rank agrees on a symmetric R-MAT graph; dropping one arc (its reversal
    kept) makes some rank refuse -- Graph.is_symmetric, exactly."""
    g0 = O.rmat_graph(1 << 12, edge_factor=8, seed=4)
    crit = P.Criterion.top_k(10, 1e-6)
    cases = [(g0.indptr, g0.indices, True)]
    cut = int(g0.indptr[7]) + 1                       # an arc of row 7
    ip = g0.indptr.copy()
    ip[8:] -= 1
    cases.append((ip, np.delete(g0.indices, cut), False))
    for ip, ix, sym in cases:
        plan = D.DevicePlan(ip.size - 1, world, int(np.diff(ip).max()))
        shards = [D.CudaShard(plan, rk, ip, ix, device=0, alpha=1e-4, gamma=1.0, crit=crit,
                              undirected=True, max_iterations=10, host_build=True)
                  for rk in range(world)]
        oks = _exchange_symmetry(shards)
        assert all(oks) == sym, (world, sym, oks)
        for s in shards:
            s.close()


def test_host_gather_shard_rejects_bad_rows():
    """Rows must hold strictly ascending ids in [0, n) (kb_graph_create's rule)."""
    g0 = O.rmat_graph(1 << 10, edge_factor=8, seed=4)
    ix = g0.indices.copy()
    ix[g0.indptr[3]], ix[g0.indptr[3] + 1] = ix[g0.indptr[3] + 1], ix[g0.indptr[3]]
    plan = D.DevicePlan(g0.node_count, 1, int(np.diff(g0.indptr).max()))
    with pytest.raises(P.ParameterError, match="ascending"):
        D.CudaShard(plan, 0, g0.indptr, ix, device=0, alpha=1e-4, gamma=1.0,
                    crit=P.Criterion.top_k(5), undirected=True, max_iterations=5,
                    host_build=True)
