#!/usr/bin/env python3
"""Benchmark: time to certified top-100 Katz ranking on R-MAT scale 24 (C2).

Contract (one JSON line on rank 0):
  step   = one certified run on the device-resident graph: init + run()
           (iterate + device check until the top-100 is certified) +
           ranking_result (order, bounds, separated fraction) kept on the
           device.  value = seconds per step (lower is better).
  e2e    = the same through the public API with HOST buffers: the canonical
           CSR is uploaded from page-locked host memory (kb_graph_create:
           H2D + device ingest), init + run, and the RankingResult arrays
           (order, lower, upper) come back to the host.
  roofline = the K1 SpMV+bounds kernel: algorithmic bytes per iteration
           B_iter = 4*nnz + w_off*(n+1) + 48*n over its
           average device duration (CUDA events on the library's stream).
  cpu_baseline = the oracle port of the reference engine on this host's
           cores, on a bounded sample (one iterate_once + check_converged on
           the full C2 graph, plus ranking_result), projected to T_cert.
  --impl reference: the reference's CPU implementation (the oracle port,
           since the reference is Python and does not travel) on the same
           config; each step = one iterate_once + check on the full graph.

Inputs are larger than L2 (2.1 GB of column ids per iteration), so no L2
flush is needed between steps.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOAD = "rmat-s24-ef16-topk100"


def workload_name(a):
    return f"rmat-s{a.scale}-ef{a.edge_factor}-topk{a.k}"
METRIC = "time to certified top-100 Katz ranking (s); GTEPS/iter; HBM GB/s vs peak"


def l2_note(nnz: int) -> str:
    return (f"inputs larger than L2: {4 * nnz / 1e9:.1f} GB of column ids streamed per "
            f"iteration (no flush needed)")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--scale", type=int, default=24)
    ap.add_argument("--edge-factor", type=int, default=16)
    ap.add_argument("--k", type=int, default=100)
    ap.add_argument("--eps", type=float, default=1e-6)
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--launcher-selftest", nargs="?", const="gloo", default=None,
                    help=argparse.SUPPRESS)
    ap.add_argument("--sharded", action="store_true",
                    help="use the row-sharded multi-GPU path even at one rank")
    ap.add_argument("--workload", default="c2", choices=["c2", "c4", "c5"],
                    help="c2: R-MAT s24 top-100 (the headline); c4: grid 4096^2 "
                         "ranking(1e-9); c5: dynamic insertion batches on c2")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region: NVML
    polled every ~2 ms from a thread (a C2 timed region is ~0.1-0.2 s), with
    nvidia-smi -lms 20 as the fallback when NVML is unavailable."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"))

    def __init__(self, device: int):
        vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
        ids = [x for x in vis.split(",") if x.strip()]
        self.device = int(ids[device]) if device < len(ids) and ids[device].isdigit() else device
        self.rows = []          # (sm_mhz, max_mhz, set of reasons)
        self.proc = None
        self.nvml = None
        self.stop = False

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nvml = nv
            self.h = nv.nvmlDeviceGetHandleByIndex(self.device)
            self.t = threading.Thread(target=self._poll, daemon=True)
            self.t.start()
            return self
        except Exception:
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device),
                 "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _poll(self):
        nv = self.nvml
        mx = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
        while not self.stop:
            sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
            bits = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            reasons = {name for name, attr in self.REASONS if bits & getattr(nv, attr)}
            self.rows.append((float(sm), float(mx), reasons))
            time.sleep(0.002)

    def _read(self):
        for line in self.proc.stdout:
            r = [x.strip() for x in line.split(",")]
            if len(r) >= 7 and r[0].replace(".", "").isdigit():
                reasons = {name for (name, _), v in zip(self.REASONS, r[3:7])
                           if v.lower() == "active"}
                self.rows.append((float(r[0]), float(r[1]), reasons))

    def __exit__(self, *a):
        self.stop = True
        if self.nvml is not None:
            self.t.join(timeout=1)
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm = sorted(r[0] for r in self.rows)
        reasons = set()
        for r in self.rows:
            reasons |= r[2]
        return {"sm_mhz": sm[len(sm) // 2] if sm else None,
                "sm_max_mhz": max(r[1] for r in self.rows) if self.rows else None,
                "reasons": sorted(reasons), "samples": len(self.rows),
                "source": "nvml" if self.nvml is not None else "nvidia-smi"}


def b_iter(n: int, nnz: int) -> int:
    w_off = 4 if nnz < 2**31 else 8
    return 4 * nnz + w_off * (n + 1) + 48 * n


def cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    import platform
    return platform.processor() or "unknown"


def port_tcert(g0, k, eps, threads):
    """One certified run of the oracle port of the reference engine --
    engine.init + engine.run (iterate_once + the reference's own
    argpartition check until certified) + ranking_result -- on `threads`
    host threads for the matvec (engine.py:181-219).  Returns (seconds,
    iterations, top-10).  Nothing is projected or extrapolated."""
    from oracle import katz_oracle as O
    t0 = time.perf_counter()
    st = O.OracleState(g0, O.Crit("topk", eps, k=k), threads=threads)
    res = O.run_reference_path(st, g0)
    return time.perf_counter() - t0, res.iterations_used, res.top(10)


def reference_package_tcert(g0, k, eps, threads):
    """The reference package itself (baseline/_ref, pip-installed from
    /root/reference; it travels to the GPU box with the snapshot) through
    the CSR shim of SURVEY.md 8(c): katzbounds.init + katzbounds.run, timed
    as cli.py:212-214 times it.  None when baseline/_ref is absent."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "katzbounds")):
        return None
    import numpy as np
    from scipy import sparse
    if ref not in sys.path:
        sys.path.insert(0, ref)
    import katzbounds as K

    class CSRShim:
        """Duck-typed static graph (engine.py:98,189,257,263,270,302); the
        arc set is the R-MAT generator's symmetric one (device-verified)."""
        node_count = g0.node_count
        version = 1

        def max_out_degree(self):
            return g0.max_out_degree()

        def is_symmetric(self):
            return True

        def out_csr(self):
            if not hasattr(self, "_csr"):
                self._csr = sparse.csr_matrix((np.ones(g0.nnz), g0.indices, g0.indptr),
                                              shape=(g0.node_count,) * 2)
            return self._csr

    g = CSRShim()
    g.out_csr()                                  # the reference caches it per version
    t0 = time.perf_counter()
    st = K.init(g, K.Criterion.top_k(k, eps), undirected=True, threads=threads)
    res = K.run(st, g)
    dt = time.perf_counter() - t0
    return {"value": dt, "unit": "s", "threads": threads, "iterations": res.iterations_used,
            "top10": [int(v) for v in res.order[:10]],
            "what": "katzbounds.init + katzbounds.run (incl. ranking_result) from baseline/_ref "
                    "through the CSR shim, out_csr() built before timing"}


def run_reference(a, rank, world):
    """--impl reference: the reference's CPU path on this host's cores.  Each
    step is one full certified run of the oracle port (r iterations of
    iterate_once + the reference's argpartition check, then ranking_result)
    with the matvec on every host thread -- measured, not projected.  Extra,
    measured once after the timed steps: the same at threads=1, and the
    reference package itself when baseline/_ref is present."""
    if rank != 0:
        return
    from oracle import katz_oracle as O
    n = 1 << a.scale
    t0 = time.perf_counter()
    g0 = O.rmat_graph(n, edge_factor=a.edge_factor, seed=a.seed)
    t_gen = time.perf_counter() - t0
    threads = os.cpu_count() or 1
    per, r_seen, top = [], None, None
    for i in range(a.warmup + a.steps):
        dt, r_seen, top = port_tcert(g0, a.k, a.eps, threads)
        if i >= a.warmup:
            per.append(dt)
    value = sum(per) / len(per)
    one_thread = None
    if not a.no_cpu:
        dt1, _, _ = port_tcert(g0, a.k, a.eps, 1)
        one_thread = {"value": dt1, "unit": "s", "cores": 1, "kind": "port",
                      "sample": "one full certified run at threads=1"}
    pkg = None
    if not a.no_cpu and os.environ.get("KB_REF_PACKAGE", "1") == "1":
        try:
            pkg = reference_package_tcert(g0, a.k, a.eps, threads)
        except Exception as e:          # noqa: BLE001 -- report, do not fail the arm
            pkg = {"error": f"{type(e).__name__}: {e}"}
    cfg = {"workload": workload_name(a), "n": n, "nnz": g0.nnz, "k": a.k, "eps": a.eps,
           "seed": a.seed, "iterations": r_seen, "max_out_degree": g0.max_out_degree(),
           "l2": l2_note(g0.nnz), "parallelism": "single"}
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "s",
        "n_gpus": world, "steps": a.steps, "warmup": a.warmup,
        "ms_per_step": value * 1e3, "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": cfg,
        "cpu_baseline": {"value": value, "unit": "s", "cores": threads, "kind": "port",
                         "sample": f"{a.steps} full certified runs (init + run to the top-{a.k} "
                                   f"certificate + ranking_result), each timed whole",
                         "cpu_model": cpu_model(), "threads_1": one_thread,
                         "reference_package": pkg},
        "e2e": {"value": value, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gteps_per_iter": None, "top10": top, "generate_s": t_gen,
    }
    print(json.dumps(line), flush=True)


def run_grid(a, device):
    """C4: grid 4096^2, Ranking(eps=1e-9) -- many iterations, deg <= 4."""
    import paper_1807_03847_b200 as P
    from paper_1807_03847_b200 import _lib
    from paper_1807_03847_b200 import generators as G
    L = _lib.lib()
    n = 1 << a.scale
    g = G.grid_graph(n, device=device)
    crit = P.Criterion.ranking(1e-9)
    nnz = int(g.device_graph.info().nnz)
    infos = []

    def step():
        st = P.init(g, crit, undirected=True, device=device, max_iterations=2000)
        out = P.engine.ctypes.c_int()
        _lib.check(L.kb_run(st._h, P.engine.ctypes.byref(out)))
        pairs = P.engine.ctypes.c_int64()
        _lib.check(L.kb_result(st._h, None, None, None, P.engine.ctypes.byref(pairs)))
        infos.append((st._info(), int(pairs.value)))

    for _ in range(a.warmup):
        step()
    ms = P.engine.ctypes.c_double()
    lc0, lc1 = P.engine.ctypes.c_int64(), P.engine.ctypes.c_int64()
    with ClockSampler(device) as clk:
        _lib.check(L.kb_launch_count(P.engine.ctypes.byref(lc0)))
        _lib.check(L.kb_timer(device, 0, None))
        for _ in range(a.steps):
            step()
        _lib.check(L.kb_timer(device, 1, P.engine.ctypes.byref(ms)))
        _lib.check(L.kb_launch_count(P.engine.ctypes.byref(lc1)))
    timed = infos[a.warmup:]
    r = int(timed[0][0].r)
    k1 = sum(i.spmv_ms for i, _ in timed) / max(1, sum(i.spmv_launches for i, _ in timed))
    # RANKING runs leave lower/upper to a lazy pass (materialize_bounds), so
    # K1 moves B_iter minus the 16 B/row of bound stores
    B = b_iter(n, nnz) - 16 * n
    peak, src = measured_peaks()
    line = {"metric": "time to certified epsilon-ranking (s)", "value": ms.value / a.steps / 1e3,
            "unit": "s", "n_gpus": 1, "steps": a.steps, "warmup": a.warmup,
            "ms_per_step": ms.value / a.steps, "higher_is_better": False, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"grid-{int(n**0.5)}x{int(n**0.5)}-ranking1e-9", "n": n,
                       "nnz": nnz, "iterations": r,
                       "separated_fraction": timed[0][1] / (n * (n - 1) // 2),
                       "full_sort_checks": int(timed[0][0].check_full_sorts)},
            "roofline": {"bound": "hbm", "achieved": B / (k1 * 1e-3) / 1e9, "peak": peak,
                         "unit": "GB/s", "frac": B / (k1 * 1e-3) / 1e9 / peak,
                         "avg_launch_ms": k1, "bytes_per_launch": B, "peak_source": src,
                         "bytes_note": "4 nnz + 4 (n+1) + 32 n: the bound stores (16 n) are "
                                       "deferred to materialize_bounds (4 passes per run)"},
            "gpu_launches": int(lc1.value - lc0.value),
            "clocks": clk.summary()}
    print(json.dumps(line), flush=True)


def run_dynamic(a, device):
    """C5: cumulative insertion batches of 1e2..1e5 undirected edges on C2
    (np.random.default_rng(7), endpoints with degree+1 < deg_max, SURVEY
    8(d)); each timed through update_batch against a static recompute."""
    import numpy as np

    import paper_1807_03847_b200 as P
    from paper_1807_03847_b200 import _lib
    from paper_1807_03847_b200 import generators as G
    L = _lib.lib()
    n = 1 << a.scale
    crit = P.Criterion.top_k(a.k, a.eps)
    if a.warmup > 0:
        # warm-up on a throwaway copy: the first update grows the device
        # memory pool (slack CSR, repair buffers); later updates reuse it
        gw = G.rmat_graph(n, edge_factor=a.edge_factor, seed=a.seed, device=device)
        sw = P.init(gw, crit, undirected=True, device=device, max_iterations=200)
        P.run(sw, gw)
        dw = gw.out_degrees()
        rw = np.random.default_rng(1234)
        cand = rw.integers(0, n, size=(4000, 2))
        cand = cand[(cand[:, 0] != cand[:, 1]) & (dw[cand[:, 0]] < 8) & (dw[cand[:, 1]] < 8)]
        cand = np.unique(np.sort(cand, axis=1), axis=0)
        cand = cand[~gw._present(cand)]
        wa = np.concatenate([cand, cand[:, ::-1]])
        P.update_batch(sw, gw, P.EdgeBatch(insertions=[tuple(x) for x in wa.tolist()]))
        P.run(P.init(gw, crit, undirected=True, device=device, max_iterations=200), gw)
        del sw, gw
        import gc
        gc.collect()             # states hold reference cycles: free the copy now
    g = G.rmat_graph(n, edge_factor=a.edge_factor, seed=a.seed, device=device)
    st = P.init(g, crit, undirected=True, device=device, max_iterations=200)
    P.run(st, g)
    deg = g.out_degrees()
    dmax = int(deg.max())
    rng = np.random.default_rng(7)
    rows = []
    for b in (100, 1000, 10000, 100000):
        picked = set()
        while len(picked) < b:
            cand = rng.integers(0, n, size=(2 * (b - len(picked)) + 16, 2))
            for u, v in cand.tolist():
                if u == v:
                    continue
                u, v = (u, v) if u < v else (v, u)
                if (u, v) in picked or deg[u] + 1 >= dmax or deg[v] + 1 >= dmax:
                    continue
                picked.add((u, v))
                if len(picked) == b:
                    break
        pk = np.array(sorted(picked), dtype=np.int64)
        pres = g._present(pk)
        pk = pk[~pres]
        arcs = np.concatenate([pk, pk[:, ::-1]])
        batch = P.EdgeBatch(insertions=arcs)          # (m, 2) int64, no tuples
        ms = P.engine.ctypes.c_double()
        _lib.check(L.kb_timer(device, 0, None))
        t0 = time.perf_counter()
        P.update_batch(st, g, batch)
        t_dyn = time.perf_counter() - t0
        _lib.check(L.kb_timer(device, 1, P.engine.ctypes.byref(ms)))
        top_dyn = P.ranking_result(st).top(a.k)
        # static recompute on the post-batch graph, best of two (the first
        # can include one-off allocations)
        t_static, ms2 = None, P.engine.ctypes.c_double()
        for _rep in range(2):
            _lib.check(L.kb_timer(device, 0, None))
            t0 = time.perf_counter()
            fres = P.run(P.init(g, crit, undirected=True, device=device, max_iterations=200), g)
            t1 = time.perf_counter() - t0
            m = P.engine.ctypes.c_double()
            _lib.check(L.kb_timer(device, 1, P.engine.ctypes.byref(m)))
            if t_static is None or t1 < t_static:
                t_static, ms2 = t1, m
        s = st.last_update_stats
        np.add.at(deg, arcs[:, 0], 1)
        rows.append({"batch_edges": int(pk.shape[0]), "update_s": t_dyn,
                     "update_device_ms": ms.value, "static_recompute_s": t_static,
                     "static_device_ms": ms2.value, "same_topk": top_dyn == fres.top(a.k),
                     "r": st.r, "level_sizes": s.level_sizes, "aborted_level": s.aborted_level,
                     "visited": s.visited, "reactivated": s.reactivated,
                     "resumed_iterations": s.resumed_iterations})
    print(json.dumps({"metric": "dynamic update vs static recompute (s)",
                      "config": {"workload": f"rmat-s{a.scale}-ef{a.edge_factor}-topk{a.k}"
                                             "-insertion-batches", "seed_batches": 7},
                      "batches": rows}), flush=True)


def shared_host_csr(g, rank, n, nnz, dist):
    """The canonical CSR in host memory once per node: rank 0 downloads it
    from its device graph into /dev/shm, the other ranks map the same pages.
    If /dev/shm cannot hold it, every rank downloads its own copy."""
    import numpy as np
    import torch
    tag = os.environ.get("MASTER_PORT", "0")
    paths = [f"/dev/shm/kb_bench_{tag}_indptr", f"/dev/shm/kb_bench_{tag}_indices"]
    ok = 1
    if rank == 0:
        try:
            ip, ix = g.csr_arrays()
            for path, arr in zip(paths, (ip, ix)):
                mm = np.lib.format.open_memmap(path, mode="w+", dtype=arr.dtype, shape=arr.shape)
                mm[:] = arr
                mm.flush()
                del mm
        except OSError:
            ok = 0
    flag = torch.tensor([ok], dtype=torch.int32, device="cuda")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    if not int(flag.item()):
        if rank == 0:
            for path in paths:
                if os.path.exists(path):
                    os.unlink(path)
        return g.csr_arrays()
    ip = np.load(paths[0], mmap_mode="r+")
    ix = np.load(paths[1], mmap_mode="r+")
    assert ip.shape == (n + 1,) and ix.shape == (nnz,)
    dist.barrier()
    if rank == 0:
        for path in paths:
            os.unlink(path)        # the mappings stay valid until closed
    return ip, ix


def run_sharded(a, rank, world, local):
    """C2 (or --scale 27: C3) on N GPUs: rows dealt by degree rank, each
    rank's shard cut out on its own GPU from the device graph
    (kb_graph_create_shard), omega exchanged every iteration by K1's fused
    NVLink stores (CUDA IPC) or an NCCL all-gather.  Strong scaling: the same
    graph at every N."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1807_03847_b200 as P
    from paper_1807_03847_b200 import _lib
    from paper_1807_03847_b200 import distributed as D
    from paper_1807_03847_b200 import generators as G
    torch.cuda.set_device(local)
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29577")
        os.environ.setdefault("RANK", str(rank))
        os.environ.setdefault("WORLD_SIZE", str(world))
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    L = _lib.lib()
    n = 1 << a.scale
    crit = P.Criterion.top_k(a.k, a.eps)
    fused = os.environ.get("KB_FUSED_EXCHANGE", "1") == "1"
    # the synthetic input: the graph generated on this rank's device
    t0 = time.perf_counter()
    gfull = G.rmat_graph(n, edge_factor=a.edge_factor, seed=a.seed, device=local)
    t_gen = time.perf_counter() - t0
    info = gfull.device_graph.info()
    nnz, d = int(info.nnz), int(info.max_out_degree)
    alpha = 1.0 / (1.0 + d)
    gamma = P.tail_gamma(alpha, d)
    plan = D.DevicePlan(n, world, d)
    split = D.fast_split(world)

    def make_shard(fz, full):
        return D.CudaShard(plan, rank, device=local, alpha=alpha, gamma=gamma, crit=crit,
                           undirected=True, max_iterations=200, split_threshold=split,
                           fused=fz, full=full)
    t0 = time.perf_counter()
    shard, exch_mode = D.connect_shard(lambda fz: make_shard(fz, gfull.device_graph), dist,
                                       rank, world, f"cuda:{local}", fused)
    shard.collective_device = f"cuda:{local}"
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t0
    shard_nnz = int(shard_info(shard).nnz)
    host_csr = None if a.no_e2e else shared_host_csr(gfull, rank, n, nnz, dist)
    gfull.device_graph.close()
    del gfull

    def step(host):
        shard.reset(alpha=alpha, gamma=gamma, crit=crit, undirected=True, max_iterations=200)
        return D.ShardedRun(shard, plan, crit, rank=rank, world=world,
                            max_iterations=200).run(host_result=host)

    # warm-up returns the ranked vectors to the host (top-10 for the line);
    # the timed steps leave them on the device like the single-GPU step
    for _ in range(a.warmup):
        res = step(True)
    dist.barrier()
    torch.cuda.synchronize()
    ms = P.engine.ctypes.c_double()
    lc0 = P.engine.ctypes.c_int64()
    _lib.check(L.kb_launch_count(P.engine.ctypes.byref(lc0)))
    with ClockSampler(local) as clk:
        _lib.check(L.kb_timer(local, 0, None))
        for _ in range(a.steps):
            r_it, _pairs = step(False)
        torch.cuda.synchronize()
        _lib.check(L.kb_timer(local, 1, P.engine.ctypes.byref(ms)))
    assert r_it == res.iterations_used
    lc1 = P.engine.ctypes.c_int64()
    _lib.check(L.kb_launch_count(P.engine.ctypes.byref(lc1)))
    k1_ms, k1_n = shard.k1_times()       # K1 launches of the last timed step
    t = torch.tensor([ms.value], device=f"cuda:{local}", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t.item()) / a.steps

    # roofline of this rank's K1 (its rows: n_per, its arcs)
    w_off = 4 if shard_nnz < 2**31 else 8
    b_rank = 4 * shard_nnz + w_off * (plan.n_per + 1) + 48 * plan.n_per
    k1_avg = k1_ms / max(1, k1_n)
    peak, peak_src = measured_peaks()
    ach = b_rank / (k1_avg * 1e-3) / 1e9 if k1_avg > 0 else 0.0
    roof = torch.tensor([ach, k1_avg], device=f"cuda:{local}", dtype=torch.float64)
    dist.all_reduce(roof, op=dist.ReduceOp.MIN)   # the slowest rank's kernel
    shard.close()

    # e2e through the public API (distributed.sharded_run) from the node's
    # host CSR; the partitioning and the symmetry check are inside the timed
    # region.
    e2e = None
    if host_csr is not None:
        ip, ix = host_csr
        for arr in (ip, ix):
            _lib.check(L.kb_host_register(_lib.ptr(arr), arr.nbytes))

        def e2e_step():
            return D.sharded_run(ip, ix, crit, undirected=True, device=local,
                                 fused=exch_mode.startswith("fused"), max_iterations=200)

        e2e_step()
        dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(a.e2e_steps):
            out = e2e_step()
        torch.cuda.synchronize()
        wall = torch.tensor([(time.perf_counter() - t0) / a.e2e_steps], device=f"cuda:{local}",
                            dtype=torch.float64)
        dist.all_reduce(wall, op=dist.ReduceOp.MAX)
        assert out.top(10) == res.top(10)
        # bytes: one rank uploads the whole CSR; more ranks upload indptr and
        # their own rows each (sharded_run's host-gather route)
        h2d = (ip.nbytes + ix.nbytes) if world == 1 else world * ip.nbytes + ix.nbytes
        e2e = {"value": float(wall.item()), "unit": "s",
               "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(world * n * 24),
               "timing": "host wall clock, max over ranks, of distributed.sharded_run from the "
                         "node's page-locked host CSR: upload (one rank: the whole CSR, the "
                         "shard cut on the device; more: indptr and the rank's own rows, "
                         "symmetry checked across ranks), run, and the ranked result "
                         "(order, lower, upper) on every rank's host"}
        for arr in (ip, ix):
            L.kb_host_unregister(_lib.ptr(arr))
    if rank == 0:
        print(json.dumps({
            "metric": METRIC, "value": ms_step / 1e3, "unit": "s", "n_gpus": world,
            "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms_step,
            "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": workload_name(a), "n": n, "nnz": nnz, "k": a.k, "eps": a.eps,
                       "seed": a.seed, "iterations": res.iterations_used,
                       "max_out_degree": d, "l2": l2_note(nnz),
                       "parallelism": f"row-shard{world}",
                       "exchange": exch_mode, "nccl_ranks": world,
                       "top10": res.top(10)},
            "gteps_per_iter": nnz * res.iterations_used / (ms_step * 1e-3) / 1e9,
            "gpu_launches": int(lc1.value - lc0.value), "clocks": clk.summary(),
            "generate_s": t_gen, "setup_s": t_setup, "e2e": e2e, "cpu_baseline": None,
            "roofline": {"bound": "hbm", "achieved": float(roof[0].item()), "peak": peak,
                         "unit": "GB/s", "frac": float(roof[0].item()) / peak, "traffic": None,
                         "kernel": "k_sell_iterate (+k_heavy_combine), per rank, slowest rank",
                         "bytes_per_launch": int(b_rank), "avg_launch_ms": float(roof[1].item()),
                         "peak_source": peak_src}}), flush=True)
    dist.barrier()
    dist.destroy_process_group()


def shard_info(shard):
    import ctypes

    from paper_1807_03847_b200 import _lib
    info = _lib.GraphInfo()
    _lib.check(shard.L.kb_graph_info_get(shard.g, ctypes.byref(info)))
    return info


def launch(a) -> int:
    """--gpus N > 1 outside torchrun: re-run this script as N ranks
    (torch.distributed.run, one process per GPU, rendezvous on 127.0.0.1).
    Fails (exit 2) if fewer than N devices are visible."""
    import socket
    if a.launcher_selftest is None and a.impl != "reference":
        import torch
        have = torch.cuda.device_count()
        if have < a.gpus:
            print(json.dumps({"error": f"--gpus {a.gpus} but only {have} CUDA devices "
                                       "are visible"}), flush=True)
            return 2
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={a.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def launcher_selftest(a, rank, world):
    """The launcher's plumbing without GPUs (CPU tests): every rank joins a
    gloo group, checks world == --gpus and all-reduces its rank."""
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo")
    t = torch.tensor([float(rank)])
    dist.all_reduce(t)
    ok = dist.get_world_size() == world == a.gpus
    if rank == 0:
        print(json.dumps({"launcher": "ok" if ok else "bad", "world": world,
                          "rank_sum": float(t.item())}), flush=True)
    dist.destroy_process_group()


def main():
    a = parse()
    rank, world, local = dist_env()
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(launch(a))
    if "WORLD_SIZE" in os.environ and world != a.gpus:
        print(json.dumps({"error": f"WORLD_SIZE={world} but --gpus {a.gpus}"}), flush=True)
        sys.exit(2)
    if a.launcher_selftest is not None:
        return launcher_selftest(a, rank, world)
    if a.impl == "reference":
        return run_reference(a, rank, world)
    if a.workload == "c4":
        if a.scale == 24:
            pass
        return run_grid(a, local)
    if a.workload == "c5":
        return run_dynamic(a, local)
    if world > 1 or a.sharded:
        return run_sharded(a, rank, world, local)

    import numpy as np

    import paper_1807_03847_b200 as P
    from paper_1807_03847_b200 import _lib
    from paper_1807_03847_b200 import generators as G

    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    device = local
    L = _lib.lib()
    n = 1 << a.scale

    t0 = time.perf_counter()
    g = G.rmat_graph(n, edge_factor=a.edge_factor, seed=a.seed, device=device)
    t_gen = time.perf_counter() - t0
    info = g.device_graph.info()
    nnz = int(info.nnz)
    crit = P.Criterion.top_k(a.k, a.eps)

    k1_times = []

    def step():
        st = P.init(g, crit, undirected=True, device=device, max_iterations=200)
        out = P.engine.ctypes.c_int()
        _lib.check(L.kb_run(st._h, P.engine.ctypes.byref(out)))
        pairs = P.engine.ctypes.c_int64()
        _lib.check(L.kb_result(st._h, None, None, None, P.engine.ctypes.byref(pairs)))
        k1_times.append(st._info())  # K1 event times (read after the step ends)
        return int(pairs.value)

    def barrier():
        if dist is not None:
            dist.barrier()

    for _ in range(a.warmup):
        step()
    lc0 = P.engine.ctypes.c_int64()
    _lib.check(L.kb_launch_count(P.engine.ctypes.byref(lc0)))
    barrier()
    ms = P.engine.ctypes.c_double()
    with ClockSampler(device) as clk:
        _lib.check(L.kb_timer(device, 0, None))
        for _ in range(a.steps):
            step()
        _lib.check(L.kb_timer(device, 1, P.engine.ctypes.byref(ms)))
    lc1 = P.engine.ctypes.c_int64()
    _lib.check(L.kb_launch_count(P.engine.ctypes.byref(lc1)))
    elapsed_ms = ms.value
    if dist is not None:
        import torch
        t = torch.tensor([elapsed_ms], device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms = float(t.item())
    ms_per_step = elapsed_ms / a.steps
    timed = k1_times[a.warmup:]
    r = int(timed[0].r)
    spmv_ms = sum(si.spmv_ms for si in timed)
    spmv_n = sum(si.spmv_launches for si in timed)
    k1_ms = spmv_ms / max(1, spmv_n)
    B = b_iter(n, nnz)
    peak, peak_src = measured_peaks()
    achieved = B / (k1_ms * 1e-3) / 1e9
    traffic = None
    gather = None
    name = "k1_traffic.json" if a.scale == 24 else f"k1_traffic_s{a.scale}.json"
    prof = os.path.join(ROOT, "profiles", name)
    if os.path.exists(prof) and a.edge_factor == 16:
        with open(prof) as fh:
            pj = json.load(fh)
        traffic = pj.get("traffic_bytes_per_launch")
        # gather-sector efficiency from the same ncu capture: the 8-byte
        # omega values the global gathers deliver over the 32-byte sectors
        # they fetch (the column stream's sectors taken out); gathers that
        # hit K1's shared-memory hot set are the arcs into its `hot` hottest
        # ids: the sum of the largest degrees
        sec = pj.get("l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", {}).get("value")
        if sec:
            stream_sectors = 4 * nnz / 32
            deg = np.sort(g.out_degrees())[::-1]
            shared_gathers = int(deg[:int(info.hot_size)].sum())
            useful = 8 * (nnz - shared_gathers)
            fetched = 32 * (sec - stream_sectors)
            gather = {"sector_efficiency": useful / fetched if fetched > 0 else None,
                      "global_gather_sectors": int(sec - stream_sectors),
                      "hot_set_gathers": shared_gathers,
                      "source": f"profiles/{name} (ncu, one K1 launch)"}
    floor = os.path.join(ROOT, "profiles", "r02_k1_c2_gather_floor.json")
    if gather is not None and a.scale == 24 and os.path.exists(floor):
        # the unit that binds K1: each 8-byte gather that misses L1 is one
        # 32-byte sector request over the L1->XBAR interface (ncu source and
        # raw pages, one K1 launch)
        with open(floor) as fh:
            fj = json.load(fh)
        mt = fj["metrics"]
        gather["binding_unit"] = {
            "unit": "L1->XBAR sector requests per SM-cycle",
            "achieved": fj["floor"]["miss_requests_per_sm_cycle"],
            "busy_frac": float(mt["l1tex__m_l1tex2xbar_req_cycles_active.avg."
                                  "pct_of_peak_sustained_elapsed"]) / 100.0,
            "source": "profiles/r02_k1_c2_gather_floor.json"}

    # ---- e2e through the public API with host buffers
    e2e = None
    if not a.no_e2e:
        indptr, indices = g.csr_arrays()
        indptr = np.ascontiguousarray(indptr)
        indices = np.ascontiguousarray(indices)
        _lib.check(L.kb_host_register(_lib.ptr(indptr), indptr.nbytes))
        _lib.check(L.kb_host_register(_lib.ptr(indices), indices.nbytes))
        order = np.empty(n, dtype=np.int64)
        lo = np.empty(n, dtype=np.float64)
        up = np.empty(n, dtype=np.float64)
        for arr in (order, lo, up):
            _lib.check(L.kb_host_register(_lib.ptr(arr), arr.nbytes))

        def e2e_step():
            dg = P.DeviceGraph(indptr, indices, device=device)
            hg = G.DeviceResidentGraph(dg)
            st = P.init(hg, crit, undirected=True, device=device, max_iterations=200)
            out = P.engine.ctypes.c_int()
            _lib.check(L.kb_run(st._h, P.engine.ctypes.byref(out)))
            pairs = P.engine.ctypes.c_int64()
            _lib.check(L.kb_result(st._h, _lib.ptr(order), _lib.ptr(lo), _lib.ptr(up),
                                   P.engine.ctypes.byref(pairs)))
            del st
            dg.close()
            return int(pairs.value)

        e2e_step()
        barrier()
        _lib.check(L.kb_timer(device, 0, None))
        t0 = time.perf_counter()
        for _ in range(a.e2e_steps):
            e2e_step()
        _lib.check(L.kb_timer(device, 1, P.engine.ctypes.byref(ms)))
        e2e_wall = (time.perf_counter() - t0) / a.e2e_steps
        e2e = {"value": e2e_wall, "unit": "s",
               "h2d_bytes_per_step": int(indptr.nbytes + indices.nbytes),
               "d2h_bytes_per_step": int(order.nbytes + lo.nbytes + up.nbytes),
               "device_ms_per_step": ms.value / a.e2e_steps,
               "timing": "host wall clock around the public calls (each ends in a "
                         "synchronising D2H copy)"}
        for arr in (indptr, indices, order, lo, up):
            L.kb_host_unregister(_lib.ptr(arr))

    # ---- CPU baseline (rank 0, N=1 only): one full certified run of the
    # reference path (oracle port) on every host core, measured whole
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu:
        from oracle import katz_oracle as O
        ip, ix = g.csr_arrays()
        g0 = O.CSRGraph(n, ip, ix, symmetric=True)
        threads = os.cpu_count() or 1
        t_cpu, r_cpu, _ = port_tcert(g0, a.k, a.eps, threads)
        cpu = {"value": t_cpu, "unit": "s", "cores": threads, "kind": "port",
               "sample": f"one full certified run (init + {r_cpu} x (iterate_once + "
                         f"argpartition check) + ranking_result) on the whole graph",
               "cpu_model": cpu_model()}

    if rank == 0:
        clocks = clk.summary()
        line = {
            "metric": METRIC,
            "value": ms_per_step / 1e3,
            "unit": "s",
            "n_gpus": world,
            "steps": a.steps,
            "warmup": a.warmup,
            "ms_per_step": ms_per_step,
            "higher_is_better": False,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": workload_name(a), "n": n, "nnz": nnz, "k": a.k,
                       "eps": a.eps, "seed": a.seed, "iterations": r,
                       "max_out_degree": int(info.max_out_degree),
                       "l2": l2_note(nnz),
                       "parallelism": "replicas" if world > 1 else "single"},
            "gteps_per_iter": nnz / (k1_ms * 1e-3) / 1e9,
            "hbm_gbs": achieved,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak,
                         "unit": "GB/s", "frac": achieved / peak, "traffic": traffic,
                         "kernel": "k_sell_iterate (+k_heavy_combine)",
                         "bytes_per_launch": B, "avg_launch_ms": k1_ms,
                         "peak_source": peak_src, "gather": gather},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(lc1.value - lc0.value),
            "clocks": clocks,
            "generate_s": t_gen,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
