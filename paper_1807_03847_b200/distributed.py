"""Multi-GPU bounded-Katz ranking: 1-D row shards and an omega all-gather.

SURVEY.md 8(e).  Rows are ranked by descending out-degree (stable in the
node id) and dealt round-robin: the row of degree rank q belongs to rank
q mod P, so every rank gets n/P rows and about nnz/P arcs.  Each rank lays its
rows out contiguously in the *exchange layout*

    e(v) = owner(v) * n_per + local(v),     n_per = ceil(n / P),

so one all-gather of every rank's block rebuilds the full omega_r replica on
every GPU.  A shard is an ordinary device graph over the exchange ids
(created with KB_GRAPH_NO_RELABEL, so its id space *is* the exchange layout)
whose non-owned rows are empty; each row keeps its arcs in the original
ascending order, so per-row sums are the single-GPU ones bit for bit.

Per iteration (run (engine.py:382-396) restated for P ranks):

  1. K1 on the local rows writes the rank's omega block;
  2. all-gather of the blocks (NCCL over NVLink);
  3. TOPK: each rank proposes its k best active nodes (key, original id,
     upper); the P*k proposals are all-gathered and every rank takes the
     same global cut and adjacent-separation test on its device
     (kb_select_global); each rank then drops its losers with the global
     threshold (kb_check_apply_cut) and |active| is all-reduced;
     SCORE: the max gap is all-reduced;
  4. ranking_result: the bound blocks are all-gathered and ranked on the
     device (kb_rank_bounds).

The collective plumbing is torch.distributed (nccl on GPUs; the CPU tests use
gloo with an oracle-backed shard).  The backend object supplies the local
compute; ``CudaShard`` is the product backend.
"""
from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _lib
from .engine import (PAIR, RANKING, SCORE, TOPK, Criterion, RankingResult,
                     default_alpha, default_iteration_cap, tail_gamma,
                     validate_alpha)
from .errors import ConvergenceError, ParameterError


class ShardPlan:
    """Degree-rank round-robin partition and the exchange layout."""

    def __init__(self, indptr: np.ndarray, nranks: int):
        if nranks < 1:
            raise ParameterError("nranks must be >= 1")
        indptr = np.asarray(indptr, dtype=np.int64)
        self.n = n = indptr.size - 1
        self.P = P = int(nranks)
        self.n_per = max(1, -(-n // P))
        deg = np.diff(indptr)
        by_rank = np.argsort(-deg, kind="stable")          # degree rank -> node
        q = np.empty(n, dtype=np.int64)
        q[by_rank] = np.arange(n, dtype=np.int64)          # node -> degree rank
        self.exch_of_node = (q % P) * self.n_per + q // P
        self.node_of_exch = np.full(P * self.n_per, -1, dtype=np.int64)
        self.node_of_exch[self.exch_of_node] = np.arange(n, dtype=np.int64)
        self.max_degree = int(deg.max()) if n else 0

    def block(self, rank: int) -> tuple[int, int]:
        return rank * self.n_per, (rank + 1) * self.n_per

    def owned(self, rank: int) -> int:
        """Rows rank owns: degree ranks q = rank (mod P) below n, laid out at
        the head of its block (the padding is the block's tail)."""
        return max(0, -(-(self.n - rank) // self.P))

    def labels(self) -> np.ndarray:
        """Tie-break labels by exchange id: the node id (padding: unique > n).
        Computed once per plan."""
        cached = getattr(self, "_labels", None)
        if cached is not None:
            return cached
        lab = self.node_of_exch.copy()
        pad = lab < 0
        lab[pad] = self.n + np.arange(int(pad.sum()))
        self._labels = lab.astype(np.int32)
        return self._labels

    def local_csr(self, indptr: np.ndarray, indices: np.ndarray, rank: int):
        """CSR over exchange ids holding only this rank's rows; each row keeps
        its original (ascending node id) order, columns mapped to exchange ids."""
        indptr = np.asarray(indptr, dtype=np.int64)
        lo, hi = self.block(rank)
        N = self.P * self.n_per
        rows = self.node_of_exch[lo:hi]
        valid = rows >= 0
        deg = np.zeros(N, dtype=np.int64)
        deg[lo:hi][valid] = indptr[rows[valid] + 1] - indptr[rows[valid]]
        ip = np.zeros(N + 1, dtype=np.int64)
        np.cumsum(deg, out=ip[1:])
        starts = indptr[rows[valid]]
        lens = deg[lo:hi][valid]
        src = np.repeat(starts - np.concatenate([[0], np.cumsum(lens)[:-1]]), lens) + \
            np.arange(int(lens.sum()), dtype=np.int64)
        ix = self.exch_of_node[np.asarray(indices)[src]].astype(np.int32)
        return ip, ix


class DevicePlan:
    """The partition of ShardPlan without its host arrays: the exchange
    layout's block sizes.  The per-node maps live on the device
    (kb_graph_create_shard)."""

    def __init__(self, n: int, nranks: int, max_degree: int):
        if nranks < 1:
            raise ParameterError("nranks must be >= 1")
        self.n, self.P = int(n), int(nranks)
        self.n_per = max(1, -(-self.n // self.P))
        self.max_degree = int(max_degree)

    block = ShardPlan.block
    owned = ShardPlan.owned


class CudaShard:
    """Product backend: this rank's shard on its GPU through the C-ABI.

    Built on the device from a device graph (``full``: an
    engine.DeviceGraph or generators.DeviceResidentGraph on this rank's GPU)
    with kb_graph_create_shard, or -- the host protocol the lockstep tests
    use -- from a ShardPlan's host CSR slice."""

    def __init__(self, plan, rank: int, indptr=None, indices=None, *, device: int,
                 alpha: float, gamma: float, crit: Criterion, undirected: bool,
                 max_iterations: int, symmetric: bool = False, split_threshold: int = 0,
                 local_csr=None, fused: bool = False, full=None, host_build: bool = False):
        import torch
        self.torch = torch
        self.L = _lib.lib()
        self.plan, self.rank, self.device = plan, rank, device
        h = ctypes.c_void_p()
        # split_threshold 0 keeps the single-GPU segmentation (2048 arcs), so
        # the shards reproduce the one-GPU bounds bit for bit; a finer split
        # (fast_split(P)) shortens the kernel tail when the per-rank work is
        # small, at the cost of rounding-level (<= 1e-12) differences
        if host_build:
            # only indptr and this rank's rows travel to its GPU
            ip = np.ascontiguousarray(indptr, dtype=np.int64)
            ix = np.ascontiguousarray(indices, dtype=np.int32)
            n_per, owned = ctypes.c_int64(), ctypes.c_int64()
            _lib.check(self.L.kb_graph_create_shard_host(
                device, ip.size - 1, int(ip[-1]), _lib.ptr(ip), _lib.ptr(ix), plan.P, rank,
                split_threshold, -1, ctypes.byref(h), ctypes.byref(n_per), ctypes.byref(owned)))
            assert (int(n_per.value), int(owned.value)) == (plan.n_per, plan.owned(rank))
        elif full is not None:
            fh = full.handle if hasattr(full, "handle") else full.device_graph.handle
            n_per, owned = ctypes.c_int64(), ctypes.c_int64()
            _lib.check(self.L.kb_graph_create_shard(fh, plan.P, rank, split_threshold, -1,
                                                    ctypes.byref(h), ctypes.byref(n_per),
                                                    ctypes.byref(owned)))
            assert (int(n_per.value), int(owned.value)) == (plan.n_per, plan.owned(rank))
        else:
            # local_csr: this rank's plan.local_csr(...) computed ahead
            ip, ix = (local_csr if local_csr is not None
                      else plan.local_csr(indptr, indices, rank))
            lab = plan.labels()
            lo, hi = plan.block(rank)
            # the symmetric flag is the caller's verified claim about the
            # whole graph (sharded_run checks it before building shards)
            flags = _lib.KB_GRAPH_NO_RELABEL | (_lib.KB_GRAPH_SYMMETRIC if symmetric else 0)
            _lib.check(self.L.kb_graph_create_ex(device, ip.size - 1, int(ip[-1]), _lib.ptr(ip),
                                                 _lib.ptr(ix), split_threshold, -1, flags,
                                                 _lib.ptr(lab), lo, hi, ctypes.byref(h)))
        self.g = h
        # fused exchange: K1 stores omega into every rank's level buffers
        # (exchange_connect); no per-iteration all-gather
        self.fused = bool(fused)
        if self.fused:
            _lib.check(self.L.kb_graph_exchange_alloc(h))
        self.reset(alpha=alpha, gamma=gamma, crit=crit, undirected=undirected,
                   max_iterations=max_iterations)

    def reset(self, *, alpha: float, gamma: float, crit: Criterion, undirected: bool,
              max_iterations: int):
        """A fresh state (engine.init) on the resident shard graph."""
        if getattr(self, "s", None):
            self.L.kb_state_destroy(self.s)
            self.s = None
        kind = {RANKING: 0, TOPK: 1, SCORE: 2, PAIR: 3}[crit.kind]
        s = ctypes.c_void_p()
        # a PAIR state's (u, v) are device ids; the sharded check reads the
        # two nodes' bounds itself (pair_values), so any distinct pair does
        pu, pv = (0, 1) if crit.kind == PAIR else (0, 0)
        _lib.check(self.L.kb_state_create(self.g, alpha, gamma, int(undirected), kind,
                                          crit.epsilon, int(crit.k or 0), pu, pv,
                                          0 if self.fused else 1, int(max_iterations),
                                          ctypes.byref(s)))
        self.s = s
        if self.fused:
            _lib.check(self.L.kb_state_exchange(s, 1))
        lo, _ = self.plan.block(self.rank)
        if crit.kind == RANKING:
            # every rank certifies the whole ranking on the gathered bounds
            _lib.check(self.L.kb_state_set_active_range(s, 0, self.plan.P * self.plan.n_per))
        else:
            _lib.check(self.L.kb_state_set_active_range(s, lo, lo + self.plan.owned(self.rank)))
        self.r = 0

    def symmetry_keys(self):
        """(keys, counts): the reverse of every local arc as an int64 device
        tensor grouped by destination rank, and the group sizes."""
        info = _lib.GraphInfo()
        _lib.check(self.L.kb_graph_info_get(self.g, ctypes.byref(info)))
        keys = self.torch.empty(max(1, int(info.nnz)), dtype=self.torch.int64,
                                device=f"cuda:{self.device}")
        counts = np.zeros(self.plan.P, dtype=np.int64)
        _lib.check(self.L.kb_shard_symmetry_keys(self.g, self.plan.P, keys.data_ptr(),
                                                 _lib.ptr(counts)))
        return keys[:int(counts.sum())], [int(c) for c in counts]

    def symmetry_verify(self, recv) -> bool:
        ok = ctypes.c_int()
        _lib.check(self.L.kb_shard_symmetry_verify(self.g, recv.data_ptr(), int(recv.numel()),
                                                   ctypes.byref(ok)))
        return bool(ok.value)

    def exchange_export(self):
        """This rank's two exchange buffers: [(ipc handle bytes, device ptr)]."""
        out = []
        for parity in (0, 1):
            hd = ctypes.create_string_buffer(64)
            _lib.check(self.L.kb_graph_exchange_handle(self.g, parity, hd))
            ptr = ctypes.c_void_p()
            _lib.check(self.L.kb_graph_exchange_ptr(self.g, parity, ctypes.byref(ptr)))
            out.append((bytes(hd.raw), int(ptr.value or 0)))
        return out

    def exchange_connect(self, exports, same_process: bool = False):
        """Register every other rank's buffers (exports[q] from rank q's
        exchange_export): opened through CUDA IPC, or used as device
        pointers when the ranks share this process."""
        for q, ex in enumerate(exports):
            if q == self.rank:
                continue
            for parity in (0, 1):
                hd, ptr = ex[parity]
                if same_process:
                    _lib.check(self.L.kb_graph_exchange_add_peer(self.g, parity, None,
                                                                 ctypes.c_void_p(ptr)))
                else:
                    buf = ctypes.create_string_buffer(hd, 64)
                    _lib.check(self.L.kb_graph_exchange_add_peer(self.g, parity, buf, None))

    def close(self):
        if getattr(self, "s", None):
            self.L.kb_state_destroy(self.s)
            self.s = None
        if getattr(self, "g", None):
            self.L.kb_graph_destroy(self.g)
            self.g = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _view(self, which: int, level: int = 0, count: int | None = None, offset: int = 0):
        ptr = ctypes.c_void_p()
        _lib.check(self.L.kb_state_vector_ptr(self.s, which, level, ctypes.byref(ptr)))
        n = count if count is not None else self.plan.P * self.plan.n_per
        iface = {"shape": (n,), "typestr": "<f8", "version": 3,
                 "data": (int(ptr.value) + 8 * offset, False)}

        class _A:
            __cuda_array_interface__ = iface
        return self.torch.as_tensor(_A(), device=f"cuda:{self.device}")

    # -- protocol
    def stream_context(self):
        """Run the collectives on the library's stream, so NCCL orders after
        the kernels that produce their inputs without a host sync."""
        if getattr(self, "_stream", None) is None:
            p = ctypes.c_void_p()
            _lib.check(self.L.kb_stream(self.device, ctypes.byref(p)))
            self._stream = self.torch.cuda.ExternalStream(int(p.value or 0),
                                                          device=f"cuda:{self.device}")
        return self.torch.cuda.stream(self._stream)

    def new_buffer(self, words: int):
        return self.torch.zeros(words, dtype=self.torch.int64, device=f"cuda:{self.device}")

    def iterate(self):
        _lib.check(self.L.kb_iterate(self.s, 1))
        self.r += 1

    def propose(self, k: int, block):
        _lib.check(self.L.kb_shard_propose(self.s, k, block.data_ptr()))

    def cut(self, blocks, nblocks: int, k: int, word):
        _lib.check(self.L.kb_shard_cut(self.s, blocks.data_ptr(), nblocks, k, word.data_ptr()))

    def commit(self, active: int):
        _lib.check(self.L.kb_shard_commit(self.s, active))

    def iterate_spec(self, word, k: int):
        """K1 of the next level behind the check's all-reduced word; it
        exits on the device if that word says converged (kb_shard_iterate_spec)."""
        _lib.check(self.L.kb_shard_iterate_spec(self.s, word.data_ptr(), k))
        self.r += 1

    def rollback(self):
        _lib.check(self.L.kb_state_rollback(self.s))
        self.r -= 1

    def level_tensor(self):
        return self._view(_lib.KB_VEC_LEVEL, self.r)

    def bounds_tensors(self):
        return self._view(_lib.KB_VEC_LOWER), self._view(_lib.KB_VEC_UPPER)

    def local_topk(self, k: int):
        keys = np.empty(k, dtype=np.uint64)
        labels = np.empty(k, dtype=np.int64)
        uppers = np.empty(k, dtype=np.float64)
        cnt = ctypes.c_int64()
        _lib.check(self.L.kb_check_local_topk(self.s, k, _lib.ptr(keys), _lib.ptr(labels),
                                              _lib.ptr(uppers), ctypes.byref(cnt)))
        c = int(cnt.value)
        return keys[:c], labels[:c], uppers[:c]

    def select_global(self, keys, labels, uppers, k: int, eps: float):
        keys = np.ascontiguousarray(keys, dtype=np.uint64)
        labels = np.ascontiguousarray(labels, dtype=np.int64)
        uppers = np.ascontiguousarray(uppers, dtype=np.float64)
        ks, ist, ok = ctypes.c_uint64(), ctypes.c_int64(), ctypes.c_int()
        _lib.check(self.L.kb_select_global(self.device, _lib.ptr(keys), _lib.ptr(labels),
                                           _lib.ptr(uppers), keys.size, k, eps, ctypes.byref(ks),
                                           ctypes.byref(ist), ctypes.byref(ok)))
        return int(ks.value), int(ist.value), bool(ok.value)

    def apply_cut(self, kstar: int, istar: int) -> int:
        m = ctypes.c_int64()
        _lib.check(self.L.kb_check_apply_cut(self.s, kstar, istar, ctypes.byref(m)))
        return int(m.value)

    def local_gap(self) -> float:
        out = ctypes.c_double()
        _lib.check(self.L.kb_gap(self.s, ctypes.byref(out)))
        return float(out.value)

    def pair_values(self, u: int, v: int):
        """(lower[u], upper[u], lower[v], upper[v]) for the nodes this rank
        owns, 0.0 for the others (an all-reduce SUM completes them)."""
        if getattr(self, "_pair_ids", None) is None or self._pair_ids[0] != (u, v):
            lab = np.array([u, v], dtype=np.int64)
            ids = np.empty(2, dtype=np.int64)
            _lib.check(self.L.kb_graph_find_labels(self.g, _lib.ptr(lab), 2, _lib.ptr(ids)))
            self._pair_ids = ((u, v), [int(x) for x in ids])
        lo, hi = self.plan.block(self.rank)
        lo_t, up_t = self.bounds_tensors()
        out = []
        for e in self._pair_ids[1]:
            own = lo <= e < hi
            out += [float(lo_t[e]) if own else 0.0, float(up_t[e]) if own else 0.0]
        return out[0], out[1], out[2], out[3]

    def check_full(self) -> bool:
        """check_converged on this rank's state, whose bounds hold every
        block (gathered): the single-GPU RANKING certificates."""
        out = ctypes.c_int()
        _lib.check(self.L.kb_check(self.s, ctypes.byref(out)))
        return bool(out.value)

    def rank_bounds(self, lower: np.ndarray, upper: np.ndarray):
        n = lower.size
        order = np.empty(n, dtype=np.int64)
        pairs = ctypes.c_int64()
        _lib.check(self.L.kb_rank_bounds(self.device, n, _lib.ptr(lower), _lib.ptr(upper),
                                         _lib.ptr(order), ctypes.byref(pairs)))
        return order, int(pairs.value)

    def rank_gathered(self, host: bool = True, out=None):
        """ranking_result of the gathered bounds, on the device: the state's
        lower/upper hold every block (exchange layout) and the graph labels
        map exchange ids to node ids (kb_rank_gathered).  host=False computes
        the order and pair count without copying the vectors back."""
        n = self.plan.n
        pairs = ctypes.c_int64()
        if not host:
            _lib.check(self.L.kb_rank_gathered(self.s, n, None, None, None, ctypes.byref(pairs)))
            return None, None, None, int(pairs.value)
        if out is not None:          # caller-provided (e.g. page-locked) arrays
            order, lower, upper = out
        else:
            order = np.empty(n, dtype=np.int64)
            lower = np.empty(n, dtype=np.float64)
            upper = np.empty(n, dtype=np.float64)
        _lib.check(self.L.kb_rank_gathered(self.s, n, _lib.ptr(order), _lib.ptr(lower),
                                           _lib.ptr(upper), ctypes.byref(pairs)))
        return order, lower, upper, int(pairs.value)

    def sync(self):
        self.torch.cuda.synchronize(self.device)

    def k1_times(self):
        """(K1 device ms summed, launches) of the current state."""
        info = _lib.StateInfo()
        _lib.check(self.L.kb_state_info_get(self.s, ctypes.byref(info)))
        return float(info.spmv_ms), int(info.spmv_launches)


def fast_split(P: int) -> int:
    """Row segmentation that keeps K1's tail short at P ranks (C2, one
    B200: P=8 rank kernel 0.60 -> 0.31 ms; profiles/r01_shard_k1_split_sweep.log)."""
    return max(512, 2048 // max(1, P))


def _all_gather_flat(dist, full, rank: int, P: int, n_per: int):
    """In-place all-gather of equal blocks of a flat tensor (one collective
    into the full buffer; the own block is staged because NCCL's in-place
    form needs the input to alias the output slot exactly)."""
    if P == 1:
        return
    mine = full[rank * n_per:(rank + 1) * n_per]
    dist.all_gather_into_tensor(full, mine)


class ShardedRun:
    """One rank's side of a sharded run (same calls on every rank)."""

    def __init__(self, backend, plan: ShardPlan, crit: Criterion, *, rank: int, world: int,
                 max_iterations: int, dist=None):
        import torch
        import torch.distributed as tdist
        self.torch = torch
        self.dist = dist or tdist
        self.b, self.plan, self.crit = backend, plan, crit
        self.rank, self.world = rank, world
        self.max_iterations = max_iterations
        if crit.kind == TOPK and crit.k > 4096:
            raise ParameterError("sharded top-k supports k <= 4096")

    def _allreduce(self, value, op):
        t = self.torch.tensor([value], dtype=self.torch.float64,
                              device=getattr(self.b, "collective_device", "cpu"))
        self.dist.all_reduce(t, op=op)
        return t.item()

    def _check(self, spec: bool = False):
        """(converged, speculated): with spec, K1 of the next level is queued
        behind the check's device word before the host reads it."""
        c = self.crit
        ops = self.dist.ReduceOp
        if c.kind == SCORE:
            return self._allreduce(self.b.local_gap(), ops.MAX) < c.epsilon, False
        if c.kind == PAIR:
            # the two nodes' bounds from their owners (engine.py:346-353)
            t = self.torch.tensor(self.b.pair_values(int(c.u), int(c.v)),
                                  dtype=self.torch.float64,
                                  device=getattr(self.b, "collective_device", "cpu"))
            self.dist.all_reduce(t, op=ops.SUM)
            lu, uu, lv, uv = t.tolist()
            u, v = int(c.u), int(c.v)
            lw, ux = (lu, uv) if (lu, -u) >= (lv, -v) else (lv, uu)
            return bool(lw > ux - c.epsilon), False
        if c.kind == RANKING:
            # every rank holds every block after the gather and runs the same
            # O(n) certificates (engine.py:355-378 with k = n): same verdict
            # on every rank, no further collective
            lo_t, up_t = self.b.bounds_tensors()
            _all_gather_flat(self.dist, lo_t, self.rank, self.plan.P, self.plan.n_per)
            _all_gather_flat(self.dist, up_t, self.rank, self.plan.P, self.plan.n_per)
            return self.b.check_full(), False
        # TOPK: fixed-size proposal blocks (count + k keys, labels, uppers as
        # 64-bit words) all-gathered on the device; every rank takes the same
        # global cut; |active| is all-reduced; one host read per check
        k = int(c.k)
        if self._blocks is None:
            self._blk = self.b.new_buffer(1 + 3 * k)
            self._blocks = self.b.new_buffer(self.world * (1 + 3 * k))
            self._word = self.b.new_buffer(3)
        self.b.propose(k, self._blk)
        self.dist.all_gather_into_tensor(self._blocks, self._blk)
        self.b.cut(self._blocks, self.world, k, self._word)
        self.dist.all_reduce(self._word[0:1], op=ops.SUM)
        spec = spec and hasattr(self.b, "iterate_spec")
        if spec:
            torch = self.torch
            if self._word_host is None:
                self._word_host = torch.empty(3, dtype=torch.int64, pin_memory=True)
                self._word_ev = torch.cuda.Event()
            self._word_host.copy_(self._word, non_blocking=True)
            self._word_ev.record()
            self.b.iterate_spec(self._word, k)     # runs while the host waits
            self._word_ev.synchronize()
            words = self._word_host.tolist()
        else:
            words = self._word.tolist()
        m_total, m_local, ok = (int(v) for v in words)
        self.b.commit(m_local)
        return m_total <= k and bool(ok), spec

    def run(self, host_result: bool = True, out=None):
        """engine.run for P ranks; every rank returns the same result.
        host_result=False leaves the ranked vectors on the device and
        returns (iterations, separated pairs) (bench timing)."""
        with self.b.stream_context():
            return self._run(host_result, out)

    def _run(self, host_result, out=None):
        P, n_per = self.plan.P, self.plan.n_per
        self._blocks = None
        self._word_host = None
        r = 0
        ahead = False                  # K1 of level r already queued
        while True:
            if not ahead:
                self.b.iterate()
            r += 1
            if not getattr(self.b, "fused", False):   # fused: K1 already stored it
                _all_gather_flat(self.dist, self.b.level_tensor(), self.rank, P, n_per)
            done, ahead = self._check(spec=r < self.max_iterations)
            if done:
                if ahead:                  # the queued K1 exited on the device
                    self.b.rollback()
                break
            if r >= self.max_iterations:
                gap = self._allreduce(self.b.local_gap(), self.dist.ReduceOp.MAX)
                raise ConvergenceError(
                    f"stopping rule still unmet after {r} iterations "
                    f"(widest bound interval {gap:.3e})", iterations=r, gap=gap)
        return self.result(r, host_result, out)

    def result(self, r: int, host: bool = True, out=None):
        P, n_per = self.plan.P, self.plan.n_per
        lo_t, up_t = self.b.bounds_tensors()
        _all_gather_flat(self.dist, lo_t, self.rank, P, n_per)
        _all_gather_flat(self.dist, up_t, self.rank, P, n_per)
        order, lower, upper, pairs = (self.b.rank_gathered(host, out=out) if out is not None
                                      else self.b.rank_gathered(host))
        if not host:
            return r, pairs
        n = self.plan.n
        for arr in (order, lower, upper):
            arr.setflags(write=False)
        frac = 1.0 if n < 2 else pairs / (n * (n - 1) // 2)
        return RankingResult(order=order, lower=lower, upper=upper, iterations_used=r,
                             criterion=self.crit, separated_fraction=frac)


def connect_shard(make_shard, dist, rank: int, world: int, device, fused: bool = True):
    """This rank's CudaShard with the fused exchange (K1 stores omega into
    every rank's level buffers through CUDA IPC mappings over NVLink) when
    all ranks can map all peers' buffers; otherwise every rank falls back to
    the per-iteration NCCL all-gather.  make_shard(fused) builds the shard.
    Returns (shard, mode)."""
    import torch
    if world == 1 or not fused:
        return make_shard(False), "nccl-allgather"
    shard, mine, err = None, None, None
    try:
        shard = make_shard(True)
        mine = shard.exchange_export()
    except Exception as e:      # noqa: BLE001 -- any failure means fall back
        err = e
    exports = [None] * world
    dist.all_gather_object(exports, mine)
    ok = all(x is not None for x in exports)
    if ok:
        try:
            shard.exchange_connect(exports)
        except Exception as e:  # noqa: BLE001
            ok, err = False, e
    flag = torch.tensor([1 if ok else 0], device=device, dtype=torch.int32)
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if int(flag.item()) == 1:
        return shard, "fused-nvlink-stores"
    if shard is not None:
        shard.close()
    return make_shard(False), f"nccl-allgather (fused exchange unavailable: {err})"


def _validate(n: int, d: int, crit: Criterion, alpha, max_iterations):
    """engine.init's checks (engine.py:248-283) for a sharded run."""
    if n < 1:
        raise ParameterError("graph must have at least one node")
    if alpha is None:
        alpha = 1.0 / (1.0 + d) if d > 0 else 0.5      # engine.py:96-99
    alpha = float(alpha)
    validate_alpha(alpha, d)
    if crit.kind == TOPK and crit.k > n:
        raise ParameterError(f"topk k={crit.k} exceeds node count {n}")
    if crit.kind == PAIR and (crit.u >= n or crit.v >= n):
        raise ParameterError("pair criterion names a node outside the graph")
    gamma = tail_gamma(alpha, d)
    if max_iterations is None:
        max_iterations = default_iteration_cap(alpha, d, crit.epsilon)
    elif max_iterations < 1:
        raise ParameterError("max_iterations must be >= 1")
    return alpha, gamma, int(max_iterations)


def shards_symmetric(shard, dist, world: int) -> bool:
    """Graph.is_symmetric (graph.py:168-175) of the sharded arc set, exactly:
    every rank sends the reverse of each of its arcs to the rank owning that
    reversed arc's row (one all-to-all), and checks that what it receives is
    exactly its own arc set; all-reduced."""
    torch = shard.torch
    dev = f"cuda:{shard.device}"
    keys, counts = shard.symmetry_keys()
    send = torch.tensor(counts, dtype=torch.int64, device=dev)
    recv_counts = torch.empty_like(send)
    dist.all_to_all_single(recv_counts, send)
    rc = [int(x) for x in recv_counts.tolist()]
    recv = torch.empty(max(1, sum(rc)), dtype=torch.int64, device=dev)[:sum(rc)]
    dist.all_to_all_single(recv, keys, output_split_sizes=rc, input_split_sizes=counts)
    ok = torch.tensor([1 if shard.symmetry_verify(recv) else 0], dtype=torch.int32, device=dev)
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    return bool(ok.item())


def sharded_run(indptr, indices, crit: Criterion, *, undirected: bool = False,
                alpha: float | None = None, max_iterations: int | None = None,
                device: int | None = None, backend_factory=None,
                fused: bool = True, graph=None) -> RankingResult:
    """engine.init + engine.run (engine.py:248-283, :382-396) of `crit` on the
    graph with the current torch.distributed group, one GPU per rank.

    The graph is the canonical CSR on every rank's host -- only indptr and
    the rank's own rows are uploaded to its GPU (kb_graph_create_shard_host,
    so graphs larger than one GPU shard too) and the arc set's symmetry is
    decided across the ranks (shards_symmetric) -- or ``graph``: a device
    graph already on this rank's GPU (engine.DeviceGraph, or a generators
    graph), cut on the device.
    undirected=True requires a symmetric arc set (ParameterError otherwise),
    as in engine.init."""
    import torch.distributed as dist
    rank, world = dist.get_rank(), dist.get_world_size()
    if backend_factory is not None:                  # host protocol (CPU tests)
        plan = ShardPlan(indptr, world)
        n, d = plan.n, plan.max_degree
        if undirected:
            ip = np.asarray(indptr, dtype=np.int64)
            rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(ip))
            cols = np.asarray(indices, dtype=np.int64)
            if not np.array_equal(np.sort(rows * n + cols), np.sort(cols * n + rows)):
                raise ParameterError("undirected mode requires a symmetric arc set")
        alpha, gamma, max_iterations = _validate(n, d, crit, alpha, max_iterations)
        backend = backend_factory(plan, rank, alpha, gamma)
        return ShardedRun(backend, plan, crit, rank=rank, world=world,
                          max_iterations=max_iterations).run()
    dev = rank if device is None else device
    own_graph = None
    if graph is None and world == 1:
        # one rank holds every row anyway: the pipelined full upload (symmetry
        # decided while the columns land) beats a host-side row gather
        from .engine import DeviceGraph
        own_graph = graph = DeviceGraph(indptr, indices, device=dev)
    if graph is not None:                           # a device graph on this rank's GPU
        dg = graph if hasattr(graph, "handle") else graph.device_graph
        info = dg.info()
        n, d = int(info.n), int(info.max_out_degree)
        alpha, gamma, max_iterations = _validate(n, d, crit, alpha, max_iterations)
        if undirected and not dg.is_symmetric():
            raise ParameterError("undirected mode requires a symmetric arc set")
        plan = DevicePlan(n, world, d)

        def make(fz):
            return CudaShard(plan, rank, device=dev, alpha=alpha, gamma=gamma, crit=crit,
                             undirected=undirected, max_iterations=max_iterations, fused=fz,
                             full=dg)
        try:
            backend, _mode = connect_shard(make, dist, rank, world, f"cuda:{dev}", fused)
        finally:
            if own_graph is not None:
                own_graph.close()
    else:
        # the host CSR: only indptr and this rank's rows go to its GPU; the
        # arc set's symmetry is then decided across the ranks, exactly
        ip = np.ascontiguousarray(indptr, dtype=np.int64)
        ix = np.ascontiguousarray(indices, dtype=np.int32)
        n = ip.size - 1
        d = int(np.diff(ip).max()) if n > 0 else 0
        alpha, gamma, max_iterations = _validate(n, d, crit, alpha, max_iterations)
        plan = DevicePlan(n, world, d)

        def make(fz):
            return CudaShard(plan, rank, ip, ix, device=dev, alpha=alpha, gamma=gamma,
                             crit=crit, undirected=undirected, max_iterations=max_iterations,
                             fused=fz, host_build=True)
        backend, _mode = connect_shard(make, dist, rank, world, f"cuda:{dev}", fused)
        if undirected and not shards_symmetric(backend, dist, world):
            backend.close()
            raise ParameterError("undirected mode requires a symmetric arc set")
    backend.collective_device = f"cuda:{dev}"
    return ShardedRun(backend, plan, crit, rank=rank, world=world,
                      max_iterations=max_iterations).run()


__all__ = ["ShardPlan", "DevicePlan", "CudaShard", "ShardedRun", "sharded_run",
           "shards_symmetric", "connect_shard", "fast_split"]
