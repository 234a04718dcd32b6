"""Dynamic edge-batch updates (katzbounds.dynamic, dynamic.py:28-211).

``update_batch`` keeps the reference's contract: all validation (batch
preconditions, undirected symmetry, post-batch alpha admission) happens
before anything mutates; then the device repairs the walk levels
(kb_update_batch, kernel K4), refreshes the bounds under the new tail
factor, reactivates nodes that may contend again, and resumes iterating
until the stopping rule holds.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .engine import KatzState, tail_gamma
from .errors import ConvergenceError, ParameterError, StateError
from .graph import EdgeBatch


@dataclass
class UpdateStats:
    """Instrumentation for one batch update (dynamic.py:28-38)."""

    batch_size: int = 0
    seeds: int = 0
    visited: int = 0
    level_sizes: list[int] = field(default_factory=list)
    reactivated: int = 0
    aborted_level: int | None = None
    resumed_iterations: int = 0


def _post_batch_max_degree(g, batch: EdgeBatch) -> int:
    """dynamic.py:152-157: max out-degree after deletions and insertions."""
    degs = np.array(g.out_degrees(), dtype=np.int64, copy=True)
    ins, dels = batch.arrays()
    if dels.shape[0]:
        np.subtract.at(degs, dels[:, 0], 1)
    if ins.shape[0]:
        np.add.at(degs, ins[:, 0], 1)
    return int(degs.max()) if degs.size else 0


def update_batch(state: KatzState, g, batch: EdgeBatch, *, theta: float = 0.5) -> None:
    """Apply an arc batch to g and bring the state back to convergence."""
    if not state.params.keep_all_levels:
        raise StateError("dynamic updates need keep_all_levels=True")
    if state.graph_version != g.version:
        raise StateError("state does not belong to this graph revision")
    if state.r < 1:
        raise StateError("run the static engine before applying updates")
    if not 0.0 <= theta <= 1.0:
        raise ParameterError(f"theta must be in [0, 1], got {theta}")
    g.validate_batch(batch)
    if state.undirected and not batch.is_symmetric():
        raise ParameterError(
            "state is in undirected mode; batch must contain both "
            "directions of every edge")
    new_max = (g.max_degree_after(batch) if hasattr(g, "max_degree_after")
               else _post_batch_max_degree(g, batch))
    if new_max > 0 and state.alpha >= 1.0 / new_max:
        raise ParameterError(
            f"batch raises max out-degree to {new_max}; alpha={state.alpha} "
            f"would leave the walk series divergent")
    new_gamma = tail_gamma(state.alpha, new_max)

    ins, dels = (np.ascontiguousarray(a) for a in batch.arrays())
    stats_c = _lib.UpdateStatsC()
    dev_version = state.device_graph.info().version
    state._touch()
    st = state._L.kb_update_batch(state._h, _lib.ptr(ins), ins.shape[0],
                                  _lib.ptr(dels), dels.shape[0], float(theta),
                                  new_gamma, ctypes.byref(stats_c))
    # the host graph follows the device (deletions then insertions,
    # dynamic.py:170, :199) whether or not the resume converged
    if st in (_lib.KB_OK, _lib.KB_ECONVERGENCE):
        if hasattr(g, "_note_device_update"):
            g._note_device_update()          # the device copy is the graph
        else:
            g.remove_arcs(batch.deletions, _validated=True)
            g.insert_arcs(batch.insertions, _validated=True)
        state.graph_version = g.version
        state.set_gamma(new_gamma)
        dg = state.device_graph
        if hasattr(g, "_device"):
            g._device = (g.version, dg)
        else:
            from .engine import _FOREIGN_CACHE
            _FOREIGN_CACHE.insert(0, (g, g.version, dg))
        stats = UpdateStats(
            batch_size=int(stats_c.batch_size), seeds=int(stats_c.seeds),
            visited=int(stats_c.visited),
            level_sizes=_level_sizes(state, stats_c),
            reactivated=int(stats_c.reactivated),
            aborted_level=None if stats_c.aborted_level < 0 else int(stats_c.aborted_level),
            resumed_iterations=int(stats_c.resumed_iterations))
        state.last_update_stats = stats
    else:
        # failed (out of memory, a CUDA error) possibly after the device had
        # applied the batch to its CSR: the state's levels may be half
        # repaired, so it refuses further use (StateError); a device copy
        # that changed no longer matches the host graph's version and is
        # dropped from every cache -- unless the device copy *is* the graph
        # (generators.DeviceResidentGraph), which then records the new arcs
        dg = state.device_graph
        if dg.info().version != dev_version:
            if hasattr(g, "_note_device_update"):
                g._note_device_update()
            else:
                _forget_device_graph(g, dg)
        state.graph_version = -1
    if st == _lib.KB_ECONVERGENCE:
        raise ConvergenceError(_lib.last_error(), iterations=state.r, gap=state.gap())
    _lib.check(st)


def _level_sizes(state: KatzState, stats_c) -> list[int]:
    """UpdateStats.level_sizes, all of it: the C struct carries the first 64."""
    n = int(stats_c.n_level_sizes)
    if n <= 64:
        return [int(x) for x in stats_c.level_sizes[:n]]
    out = np.empty(n, dtype=np.int64)
    cnt = ctypes.c_int64()
    _lib.check(state._L.kb_update_level_sizes(state._h, _lib.ptr(out), n, ctypes.byref(cnt)))
    return [int(x) for x in out[:int(cnt.value)]]


def _forget_device_graph(g, dg) -> None:
    if hasattr(g, "_device"):
        cached = g._device
        if cached is not None and cached[1] is dg:
            g._device = None
        return
    from .engine import _FOREIGN_CACHE
    _FOREIGN_CACHE[:] = [e for e in _FOREIGN_CACHE if e[2] is not dg]
