"""ctypes binding of the native engine (include/katzb200.h).

The shared library is built in-tree by ``__graft_entry__.build()`` into
``paper_1807_03847_b200/_lib/libkatzb200.so``.  There is no CPU fallback:
if the library or a CUDA device is missing, every compute entry point raises.
"""
from __future__ import annotations

import ctypes
import os

from .errors import (BatchPreconditionError, ConvergenceError, DeviceError,
                     NodeRangeError, NumericError, ParameterError, StateError)

# KB_LIB=checked loads the checked build (device invariants polled after
# every call; `make -C paper_1807_03847_b200/csrc checked`)
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)),
                        "_lib_checked" if os.environ.get("KB_LIB") == "checked" else "_lib",
                        "libkatzb200.so")

KB_OK, KB_EPARAM, KB_ESTATE, KB_ECONVERGENCE, KB_ENUMERIC = 0, 1, 2, 3, 4
KB_EBATCH, KB_ENODERANGE, KB_ECUDA, KB_ENOMEM = 5, 6, 7, 8
KB_RANKING, KB_TOPK, KB_SCORE, KB_PAIR = 0, 1, 2, 3
KB_VEC_LEVEL, KB_VEC_KATZ, KB_VEC_LOWER, KB_VEC_UPPER = 0, 1, 2, 3
KB_GRAPH_NO_RELABEL, KB_GRAPH_SYMMETRIC = 1, 2

_ERRORS = {
    KB_EPARAM: ParameterError,
    KB_ESTATE: StateError,
    KB_ENUMERIC: NumericError,
    KB_EBATCH: BatchPreconditionError,
    KB_ENODERANGE: NodeRangeError,
    KB_ECUDA: DeviceError,
    KB_ENOMEM: DeviceError,
}

i64, i32, dbl, vp = ctypes.c_int64, ctypes.c_int, ctypes.c_double, ctypes.c_void_p


class GraphInfo(ctypes.Structure):
    _fields_ = [(name, i64) for name in (
        "n", "nnz", "max_out_degree", "nonisolated", "heavy_rows", "segments",
        "slices", "sell_elems", "split_threshold", "hot_size", "version",
        "device_bytes", "overflow_rows", "overflow_long")]


class StateInfo(ctypes.Structure):
    _fields_ = [("r", i64), ("active", i64), ("max_iterations", i64),
                ("levels_kept", i64), ("alpha", dbl), ("gamma", dbl),
                ("epsilon", dbl), ("last_check_ms", dbl), ("spmv_ms", dbl),
                ("spmv_launches", i64), ("check_full_sorts", i64),
                ("k_boundary_ties", i64)]


class UpdateStatsC(ctypes.Structure):
    _fields_ = [("batch_size", i64), ("seeds", i64), ("visited", i64),
                ("reactivated", i64), ("resumed_iterations", i64),
                ("aborted_level", i64), ("n_level_sizes", i64),
                ("level_sizes", i64 * 64)]


# name -> (restype, argtypes); the set of symbols include/katzb200.h declares
SIGNATURES = {
    "kb_last_error": (ctypes.c_char_p, []),
    "kb_version": (i32, []),
    "kb_device_count": (i32, [ctypes.POINTER(i32)]),
    "kb_timer": (i32, [i32, i32, ctypes.POINTER(dbl)]),
    "kb_launch_count": (i32, [ctypes.POINTER(i64)]),
    "kb_tune": (i32, [ctypes.c_char_p, i64]),
    "kb_host_register": (i32, [vp, i64]),
    "kb_host_unregister": (i32, [vp]),
    "kb_graph_create": (i32, [i32, i64, i64, vp, vp, i64, i64, ctypes.POINTER(vp)]),
    "kb_graph_create_ex": (i32, [i32, i64, i64, vp, vp, i64, i64, i32, vp, i64, i64,
                                 ctypes.POINTER(vp)]),
    "kb_graph_find_labels": (i32, [vp, vp, i64, vp]),
    "kb_graph_create_shard_host": (i32, [i32, i64, i64, vp, vp, i64, i64, i64, i64,
                                         ctypes.POINTER(vp), ctypes.POINTER(i64),
                                         ctypes.POINTER(i64)]),
    "kb_shard_symmetry_keys": (i32, [vp, i64, vp, vp]),
    "kb_shard_symmetry_verify": (i32, [vp, vp, i64, ctypes.POINTER(i32)]),
    "kb_graph_create_shard": (i32, [vp, i64, i64, i64, i64, ctypes.POINTER(vp),
                                    ctypes.POINTER(i64), ctypes.POINTER(i64)]),
    "kb_graph_create_rmat": (i32, [i32, i32, i64, vp, dbl, dbl, dbl, i64, i64,
                                   ctypes.POINTER(vp)]),
    "kb_graph_create_grid": (i32, [i32, i64, i64, i64, ctypes.POINTER(vp)]),
    "kb_graph_get_csr": (i32, [vp, vp, vp]),
    "kb_graph_has_arcs": (i32, [vp, vp, i64, vp]),
    "kb_graph_max_degree_after": (i32, [vp, vp, i64, vp, i64, ctypes.POINTER(i64)]),
    "kb_graph_out_degrees": (i32, [vp, vp]),
    "kb_graph_apply_batch": (i32, [vp, vp, i64, vp, i64]),
    "kb_graph_destroy": (i32, [vp]),
    "kb_graph_info_get": (i32, [vp, ctypes.POINTER(GraphInfo)]),
    "kb_graph_is_symmetric": (i32, [vp, ctypes.POINTER(i32)]),
    "kb_state_create": (i32, [vp, dbl, dbl, i32, i32, dbl, i64, i64, i64, i32, i64,
                              ctypes.POINTER(vp)]),
    "kb_state_destroy": (i32, [vp]),
    "kb_state_info_get": (i32, [vp, ctypes.POINTER(StateInfo)]),
    "kb_state_set_max_iterations": (i32, [vp, i64]),
    "kb_iterate": (i32, [vp, i64]),
    "kb_check": (i32, [vp, ctypes.POINTER(i32)]),
    "kb_run": (i32, [vp, ctypes.POINTER(i32)]),
    "kb_gap": (i32, [vp, ctypes.POINTER(dbl)]),
    "kb_epsilon_separated": (i32, [vp, i64, i64, ctypes.POINTER(i32)]),
    "kb_result": (i32, [vp, vp, vp, vp, ctypes.POINTER(i64)]),
    "kb_separated_pairs": (i32, [vp, ctypes.POINTER(i64)]),
    "kb_get_vector": (i32, [vp, i32, i64, vp]),
    "kb_get_active": (i32, [vp, vp]),
    "kb_state_set_active": (i32, [vp, vp, i64]),
    "kb_state_set_active_range": (i32, [vp, i64, i64]),
    "kb_state_vector_ptr": (i32, [vp, i32, i64, ctypes.POINTER(vp)]),
    "kb_sync": (i32, [i32]),
    "kb_check_local_topk": (i32, [vp, i64, vp, vp, vp, ctypes.POINTER(i64)]),
    "kb_select_global": (i32, [i32, vp, vp, vp, i64, i64, dbl, ctypes.POINTER(ctypes.c_uint64),
                               ctypes.POINTER(i64), ctypes.POINTER(i32)]),
    "kb_check_apply_cut": (i32, [vp, ctypes.c_uint64, i64, ctypes.POINTER(i64)]),
    "kb_rank_bounds": (i32, [i32, i64, vp, vp, vp, ctypes.POINTER(i64)]),
    "kb_text_scan": (i32, [i32, vp, i64, i32, ctypes.POINTER(vp), vp]),
    "kb_text_candidates": (i32, [vp, vp]),
    "kb_text_lines": (i32, [vp, vp, vp, vp]),
    "kb_text_destroy": (i32, [vp]),
    "kb_graph_create_text": (i32, [vp, i64, i32, vp, i64, i64, i64, ctypes.POINTER(vp)]),
    "kb_foster": (i32, [vp, dbl, dbl, i64, vp, ctypes.POINTER(i64), ctypes.POINTER(dbl)]),
    "kb_cg_katz": (i32, [vp, dbl, dbl, i64, vp, ctypes.POINTER(i64), ctypes.POINTER(dbl)]),
    "kb_ranking_inversions": (i32, [i32, i64, vp, vp, ctypes.POINTER(i64)]),
    "kb_ranking_snapshot": (i32, [vp, ctypes.POINTER(vp), ctypes.POINTER(i64)]),
    "kb_ranking_read": (i32, [vp, i32, i64, i64, vp]),
    "kb_ranking_destroy": (i32, [vp]),
    "kb_pool_info": (i32, [i32, vp]),
    "kb_pool_reserve": (i32, [i32, i64]),
    "kb_stream": (i32, [i32, ctypes.POINTER(vp)]),
    "kb_shard_propose": (i32, [vp, i64, vp]),
    "kb_shard_cut": (i32, [vp, vp, i64, i64, vp]),
    "kb_shard_commit": (i32, [vp, i64]),
    "kb_shard_iterate_spec": (i32, [vp, vp, i64]),
    "kb_state_rollback": (i32, [vp]),
    "kb_rank_gathered": (i32, [vp, i64, vp, vp, vp, ctypes.POINTER(i64)]),
    "kb_graph_exchange_alloc": (i32, [vp]),
    "kb_graph_exchange_ptr": (i32, [vp, i32, ctypes.POINTER(vp)]),
    "kb_graph_exchange_handle": (i32, [vp, i32, vp]),
    "kb_graph_exchange_add_peer": (i32, [vp, i32, vp, vp]),
    "kb_state_exchange": (i32, [vp, i32]),
    "kb_update_level_sizes": (i32, [vp, vp, i64, ctypes.POINTER(i64)]),
    "kb_update_batch": (i32, [vp, vp, i64, vp, i64, dbl, dbl,
                              ctypes.POINTER(UpdateStatsC)]),
}

_lib = None


def lib():
    """Load the native library (raises loudly if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"native engine not built: {LIB_PATH} is missing; run "
                "`python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        # KB_TUNE="name=value,...": tuning knobs for experiments (tools/)
        for item in filter(None, os.environ.get("KB_TUNE", "").split(",")):
            k, _, v = item.partition("=")
            L.kb_tune(k.strip().encode(), int(v))
        _lib = L
    return _lib


def last_error() -> str:
    msg = lib().kb_last_error()
    return msg.decode() if msg else ""


def check(status: int, **conv) -> None:
    """Raise the katzbounds-style error for a non-zero status."""
    if status == KB_OK:
        return
    msg = last_error()
    if status == KB_ECONVERGENCE:
        raise ConvergenceError(msg, **conv)
    raise _ERRORS.get(status, DeviceError)(msg)


def ptr(a):
    return a.ctypes.data_as(vp)
