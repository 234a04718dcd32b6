"""The paper's method comparison (reference cli.py:293-386, cmd_compare and
concordant_fraction), without the command-line shell.

``compare`` runs the bounded engine with a full-ranking criterion next to the
Foster and CG baselines on the same device graph and returns the same
RunReport the reference's ``compare`` command emits.  ``concordant_fraction``
counts discordant pairs on the device (kb_ranking_inversions: an MSB-first
radix split, exact in 64 bits) where the reference runs a pure-Python merge
sort.
"""
from __future__ import annotations

import ctypes
import time

import numpy as np

from . import _lib
from .baselines import cg_katz, foster
from .engine import PAIR, TOPK, Criterion, init, run
from .errors import KatzError
from .reports import RunReport

DEFAULT_EPSILON = 1e-6


def ranking_inversions(order_a, order_b, *, device: int = 0) -> int:
    """Node pairs the two rankings order differently."""
    a = np.ascontiguousarray(order_a, dtype=np.int64)
    b = np.ascontiguousarray(order_b, dtype=np.int64)
    if a.shape != b.shape or a.ndim != 1:
        raise KatzError("rankings must be 1-D and of equal length")
    out = ctypes.c_int64()
    _lib.check(_lib.lib().kb_ranking_inversions(device, a.size, _lib.ptr(a), _lib.ptr(b),
                                                ctypes.byref(out)))
    return int(out.value)


def concordant_fraction(order_a, order_b, *, device: int = 0) -> float:
    """Fraction of node pairs ordered the same way by both rankings
    (cli.py:349-360)."""
    n = len(order_a)
    if n < 2:
        return 1.0
    return 1.0 - ranking_inversions(order_a, order_b, device=device) / (n * (n - 1) // 2)


def engine_parameters(state) -> dict:
    """The report's parameter block (cli.py:181-195)."""
    crit = state.criterion
    p = {"criterion": crit.kind, "epsilon": crit.epsilon, "alpha": state.alpha,
         "gamma": state.gamma, "undirected": state.undirected, "threads": state.threads}
    if crit.kind == TOPK:
        p["k"] = crit.k
    if crit.kind == PAIR:
        p["pair"] = [crit.u, crit.v]
    return p


def compare(g, *, methods: str = "katz,foster,cg", epsilon: float = DEFAULT_EPSILON,
            alpha: float | None = None, undirected: bool = False, foster_tol: float = 1e-9,
            cg_tol: float = 1e-15, threads: int | None = None, device: int = 0):
    """cmd_compare (cli.py:293-346): returns (report, result), the result
    being the bounded engine's RankingResult (for per-node output)."""
    names = [m.strip() for m in methods.split(",") if m.strip()]
    unknown = set(names) - {"katz", "foster", "cg"}
    if unknown:
        raise KatzError(f"unknown methods: {', '.join(sorted(unknown))}")
    state = init(g, Criterion.ranking(epsilon), alpha=alpha, undirected=undirected,
                 threads=threads if threads is not None else 1, device=device)
    t0 = time.perf_counter()
    result = run(state, g)
    katz_wall = time.perf_counter() - t0
    top = min(10, state.n)
    entries = [{"method": "katz-bounds", "iterations": result.iterations_used,
                "wall_time_s": katz_wall, "separated_fraction": result.separated_fraction,
                "top": result.top(top), "ranking_agreement": 1.0}]
    for name in names:
        if name == "katz":
            continue
        t0 = time.perf_counter()
        if name == "foster":
            sv = foster(g, alpha=state.alpha, tol=foster_tol, device=device)
        else:
            sv = cg_katz(g, alpha=state.alpha, residual_tol=cg_tol, device=device)
        wall = time.perf_counter() - t0
        ranking = sv.ranking()
        entries.append({"method": sv.method, "iterations": sv.iterations,
                        "residual": sv.residual, "wall_time_s": wall,
                        "top": [int(v) for v in ranking[:top]],
                        "ranking_agreement": concordant_fraction(result.order, ranking,
                                                                 device=device)})
    report = RunReport(command="compare", method="katz-bounds",
                       parameters=engine_parameters(state),
                       iterations=result.iterations_used,
                       wall_time_s=katz_wall + sum(e["wall_time_s"] for e in entries[1:]),
                       separated_fraction=result.separated_fraction,
                       ranking_prefix=result.top(top), extra={"methods": entries})
    return report, result


__all__ = ["compare", "concordant_fraction", "ranking_inversions", "engine_parameters"]
