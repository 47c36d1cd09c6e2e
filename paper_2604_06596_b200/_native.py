"""ctypes binding of libdynlp_b200.so (include/dynlp_b200.h).

The library is built in-tree (paper_2604_06596_b200/build.py) and travels
with the repository snapshot.  There is no fallback: if the library is
missing or cannot be loaded, every entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DLP_LIB_PATH") or os.path.join(HERE, "libdynlp_b200.so")


class Batch(C.Structure):
    _fields_ = [
        ("t", C.c_int64),
        ("n_ins", C.c_int64), ("insert_ids", C.c_void_p), ("insert_gt", C.c_void_p),
        ("n_edges", C.c_int64), ("edge_owner", C.c_void_p), ("edge_other", C.c_void_p),
        ("edge_w", C.c_void_p),
        ("n_del", C.c_int64), ("deletes", C.c_void_p),
    ]


class Config(C.Structure):
    _fields_ = [
        ("delta", C.c_double), ("tau", C.c_double), ("max_iterations", C.c_int64),
        ("component_init", C.c_int32), ("mode", C.c_int32), ("num_classes", C.c_int32),
        ("reserved", C.c_int32),
    ]


class Report(C.Structure):
    _fields_ = [
        ("t", C.c_int64), ("iterations", C.c_int64), ("updates", C.c_int64),
        ("max_change", C.c_double), ("converged", C.c_int32), ("pad", C.c_int32),
        ("warnings", C.c_int64), ("isolated_pinned", C.c_int64),
        ("unreachable_pinned", C.c_int64), ("wall_time_ms", C.c_double),
        ("edges_traversed", C.c_int64), ("certify_sweeps", C.c_int64),
        ("lp_kernel_ms", C.c_double), ("gpu_launches", C.c_int64), ("lp_rounds", C.c_int64),
        ("lp_union_rows", C.c_int64), ("lp_union_entries", C.c_int64),
    ]


# name -> (restype, argtypes); the exported surface of include/dynlp_b200.h
_p, _i64, _i32, _dbl, _int = C.c_void_p, C.c_int64, C.c_int32, C.c_double, C.c_int
SIGNATURES = {
    "dlp_create": (_int, [_p, _int, _p]),
    "dlp_destroy": (_int, [_p]),
    "dlp_last_error": (C.c_char_p, [_p]),
    "dlp_num_columns": (_int, [_p]),
    "dlp_apply_batch": (_int, [_p, _p, _p, _p]),
    "dlp_apply_batch_device": (_int, [_p, _p, _p, _int, _p]),
    "dlp_apply_batch_pipelined": (_int, [_p, _p, _p, _p, _p]),
    "dlp_apply_structure": (_int, [_p, _p]),
    "dlp_itlp_batch": (_int, [_p, _p, _p, _p]),
    "dlp_reserve": (_int, [_p, _i64, _i64]),
    "dlp_nccl_unique_id": (_int, [_p]),
    "dlp_shard_nccl": (_int, [_p, _p, _int, _int]),
    "dlp_shard_set": (_int, [_p, _int, _int]),
    "dlp_shard_mode": (_int, [_p, _int]),
    "dlp_apply_batch_sharded": (_int, [_p, _p, _p, _p, _p, _p]),
    "dlp_read_owned": (_int, [_p, _p, _i64]),
    "dlp_num_slots": (_int, [_p, _p, _p]),
    "dlp_read_labels": (_int, [_p, _p, _p, _i64]),
    "dlp_write_labels": (_int, [_p, _p, _i64]),
    "dlp_harmonic_solve": (_int, [_p, _int, _i64, _p, _i64, _p]),
    "dlp_read_alive": (_int, [_p, _p, _i64]),
    "dlp_read_eligible": (_int, [_p, _p, _i64]),
    "dlp_graph_stats": (_int, [_p, _p, _p]),
    "dlp_read_csr": (_int, [_p, _p, _p, _p, _p, _i64, _i64]),
    "dlp_read_live_edges": (_int, [_p, _p, _p, _p, _i64]),
    "dlp_read_intra": (_int, [_p, _p, _p, _p, _i64, _p]),
    "dlp_jacobi_step": (_int, [_p, _p, _p, _p, _p, _i64, _p, _i64, _p, _p]),
    "dlp_gauss_seidel_step": (_int, [_p, _p, _p, _p, _p, _i64, _p, _i64, _p]),
    "dlp_jacobi_run": (_int, [_p, _p, _p, _p, _p, _i64, _p, _i64, _p, _dbl, _i64,
                              _p, _p, _p, _p, _p, _p]),
    "dlp_plugin_last_error": (C.c_char_p, []),
    "dlp_knn_create": (_int, [_int, _p]),
    "dlp_knn_destroy": (_int, [_p]),
    "dlp_knn_last_error": (C.c_char_p, [_p]),
    "dlp_knn_set_features": (_int, [_p, _p, _i64, _i64]),
    "dlp_knn_query": (_int, [_p, _i64, _i64, _i32, _p, _p]),
    "dlp_knn_graph": (_int, [_p, _i32, _i32, _p]),
    "dlp_knn_read_edges": (_int, [_p, _p, _p, _p, _i64]),
    "dlp_knn_stats": (_int, [_p, _p, _p, _p, _p, _p, _p]),
    "dlp_knn_debug_candidates": (_int, [_p, _i64, _i64, _p, _p, _p, _p, _i64]),
    "dlp_device_info": (_int, [_int, _p, _p, _p]),
}

_lib = None
_lock = threading.Lock()


def load(build_if_missing: bool = False):
    """Load the native library (raises if it is absent: no CPU fallback)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            if build_if_missing:
                from . import build

                build.build()
            else:
                raise ImportError(
                    f"{LIB_PATH} is missing: build it with `python -m paper_2604_06596_b200.build` "
                    "(the B200 engine has no CPU fallback)")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            if os.environ.get("DLP_LIB_PATH") and not hasattr(lib, name):
                continue  # an older tuning variant (A/B runs) may lack newer entry points
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def ptr(a):
    return None if a is None else a.ctypes.data
