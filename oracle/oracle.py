"""ctypes binding of oracle/dynlp_oracle.c (TEST INFRASTRUCTURE ONLY)."""

from __future__ import annotations

import ctypes as C
import importlib
import math
import os
import sys
from dataclasses import dataclass

import numpy as np

from . import build as _build

_HERE = os.path.dirname(os.path.abspath(__file__))


class _Batch(C.Structure):
    _fields_ = [
        ("t", C.c_int64),
        ("n_ins", C.c_int64), ("insert_ids", C.c_void_p), ("insert_gt", C.c_void_p),
        ("n_edges", C.c_int64), ("edge_owner", C.c_void_p), ("edge_other", C.c_void_p),
        ("edge_w", C.c_void_p),
        ("n_del", C.c_int64), ("deletes", C.c_void_p),
    ]


class _Config(C.Structure):
    _fields_ = [
        ("delta", C.c_double), ("tau", C.c_double), ("max_iterations", C.c_int64),
        ("component_init", C.c_int32), ("mode", C.c_int32),
    ]


class _Report(C.Structure):
    _fields_ = [
        ("t", C.c_int64), ("iterations", C.c_int64), ("updates", C.c_int64),
        ("max_change", C.c_double), ("converged", C.c_int32), ("pad", C.c_int32),
        ("warnings", C.c_int64), ("isolated_pinned", C.c_int64),
        ("unreachable_pinned", C.c_int64), ("wall_time_ms", C.c_double),
        ("edges_traversed", C.c_int64), ("certify_sweeps", C.c_int64),
    ]


_lib = None


def _load():
    global _lib
    if _lib is None:
        path = _build.build_oracle()
        lib = C.CDLL(path)
        p, i64, i32, dbl = C.c_void_p, C.c_int64, C.c_int32, C.c_double
        sig = {
            "orc_create": (p, [i32, i32]),
            "orc_destroy": (None, [p]),
            "orc_last_error": (C.c_char_p, [p]),
            "orc_num_columns": (i32, [p]),
            "orc_apply_batch": (C.c_int, [p, p, p, p]),
            "orc_apply_structure": (C.c_int, [p, p]),
            "orc_num_slots": (i64, [p]),
            "orc_num_alive": (i64, [p]),
            "orc_num_live_edges": (i64, [p]),
            "orc_last_tau": (dbl, [p]),
            "orc_read_labels": (None, [p, p, p]),
            "orc_write_labels": (None, [p, p]),
            "orc_read_alive": (None, [p, p]),
            "orc_read_csr": (None, [p, p, p, p, p]),
            "orc_read_live_edges": (None, [p, p, p, p]),
            "orc_read_eligible": (None, [p, p]),
            "orc_intra_size": (i64, [p]),
            "orc_read_intra": (i64, [p, p, p, p]),
            "orc_pairwise_sum": (dbl, [p, i64]),
            "orc_jacobi_step": (None, [p, p, p, p, p, p, i64, p, p, i32]),
            "orc_gauss_seidel_step": (None, [p, p, p, p, p, p, i64, p]),
            "orc_jacobi_run": (i64, [p, p, p, p, p, i64, p, i64, p, dbl, i64, i32, p, p, p, p, p]),
        }
        for name, (res, args) in sig.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data


@dataclass
class OracleReport:
    t: int
    iterations: int
    updates: int
    max_change: float
    converged: bool
    warnings: int
    isolated_pinned: int
    unreachable_pinned: int
    wall_time_ms: float
    edges_traversed: int
    certify_sweeps: int


class OracleError(ValueError):
    pass


def _batch_struct(batch, keep):
    arrs = dict(
        insert_ids=np.ascontiguousarray(batch.insert_ids, dtype=np.int64),
        insert_gt=np.ascontiguousarray(batch.insert_gt, dtype=np.int8),
        edge_owner=np.ascontiguousarray(batch.edge_owner, dtype=np.int64),
        edge_other=np.ascontiguousarray(batch.edge_other, dtype=np.int64),
        edge_w=np.ascontiguousarray(batch.edge_w, dtype=np.float64),
        deletes=np.ascontiguousarray(batch.deletes, dtype=np.int64),
    )
    keep.append(arrs)
    return _Batch(
        int(batch.t), len(arrs["insert_ids"]), _ptr(arrs["insert_ids"]), _ptr(arrs["insert_gt"]),
        len(arrs["edge_owner"]), _ptr(arrs["edge_owner"]), _ptr(arrs["edge_other"]),
        _ptr(arrs["edge_w"]), len(arrs["deletes"]), _ptr(arrs["deletes"]),
    )


class OracleEngine:
    """C restatement of DynamicGraph + LabelState + apply_batch, one label
    column for binary runs, C one-vs-rest columns for C > 2 classes."""

    def __init__(self, num_classes: int = 2, threads: int = 1):
        self._lib = _load()
        self._h = self._lib.orc_create(num_classes, threads)
        self.num_classes = num_classes
        self.ncol = self._lib.orc_num_columns(self._h)

    def __del__(self):
        if getattr(self, "_h", None):
            self._lib.orc_destroy(self._h)
            self._h = None

    def apply_batch(self, batch, delta=1e-4, tau="auto", max_iterations=None,
                    component_init=True, mode="parallel_jacobi"):
        keep = []
        b = _batch_struct(batch, keep)
        cfg = _Config(float(delta), math.nan if tau == "auto" else float(tau),
                      0 if max_iterations is None else int(max_iterations),
                      1 if component_init else 0,
                      0 if mode == "parallel_jacobi" else 1)
        reps = (_Report * self.ncol)()
        rc = self._lib.orc_apply_batch(self._h, C.byref(cfg), C.byref(b), reps)
        if rc:
            raise OracleError(self._lib.orc_last_error(self._h).decode())
        return [OracleReport(r.t, r.iterations, r.updates, r.max_change, bool(r.converged),
                             r.warnings, r.isolated_pinned, r.unreachable_pinned,
                             r.wall_time_ms, r.edges_traversed, r.certify_sweeps) for r in reps]

    def apply_structure(self, batch):
        keep = []
        b = _batch_struct(batch, keep)
        rc = self._lib.orc_apply_structure(self._h, C.byref(b))
        if rc:
            raise OracleError(self._lib.orc_last_error(self._h).decode())

    @property
    def num_slots(self) -> int:
        return int(self._lib.orc_num_slots(self._h))

    @property
    def num_alive(self) -> int:
        return int(self._lib.orc_num_alive(self._h))

    @property
    def last_tau(self) -> float:
        return float(self._lib.orc_last_tau(self._h))

    def labels(self):
        n = self.num_slots
        f = np.empty((self.ncol, n), dtype=np.float64)
        gt = np.empty(n, dtype=np.int8)
        self._lib.orc_read_labels(self._h, _ptr(f), _ptr(gt))
        return f, gt

    def write_labels(self, f):
        f = np.ascontiguousarray(f, dtype=np.float64).reshape(self.ncol, self.num_slots)
        self._lib.orc_write_labels(self._h, _ptr(f))

    def alive(self):
        a = np.empty(self.num_slots, dtype=np.uint8)
        self._lib.orc_read_alive(self._h, _ptr(a))
        return a.astype(bool)

    def eligible(self):
        a = np.empty(self.num_slots, dtype=np.uint8)
        self._lib.orc_read_eligible(self._h, _ptr(a))
        return a.astype(bool)

    def csr(self):
        n = self.num_slots
        m = int(self._lib.orc_num_live_edges(self._h))
        indptr = np.empty(n + 1, dtype=np.int64)
        indices = np.empty(2 * m, dtype=np.int64)
        weights = np.empty(2 * m, dtype=np.float64)
        degrees = np.empty(n, dtype=np.float64)
        self._lib.orc_read_csr(self._h, _ptr(indptr), _ptr(indices), _ptr(weights), _ptr(degrees))
        return indptr, indices, weights, degrees

    def live_edges(self):
        m = int(self._lib.orc_num_live_edges(self._h))
        u = np.empty(m, dtype=np.int64)
        v = np.empty(m, dtype=np.int64)
        w = np.empty(m, dtype=np.float64)
        self._lib.orc_read_live_edges(self._h, _ptr(u), _ptr(v), _ptr(w))
        return u, v, w

    def intra_labeling(self):
        k = int(self._lib.orc_intra_size(self._h))
        v = np.empty(k, dtype=np.int64)
        p = np.empty(k, dtype=np.int64)
        c = np.empty(k, dtype=np.int64)
        self._lib.orc_read_intra(self._h, _ptr(v), _ptr(p), _ptr(c))
        return v, p, c


def pairwise_sum(a) -> float:
    a = np.ascontiguousarray(a, dtype=np.float64)
    return float(_load().orc_pairwise_sum(_ptr(a), len(a)))


def _c64(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


def orc_jacobi_step(indptr, indices, weights, gt, f, frontier, out_vals, out_deltas, threads=1):
    args = [_c64(indptr, np.int64), _c64(indices, np.int64), _c64(weights, np.float64),
            _c64(gt, np.int8), _c64(f, np.float64), _c64(frontier, np.int64)]
    _load().orc_jacobi_step(*[_ptr(a) for a in args[:6]], len(args[5]), _ptr(out_vals),
                            _ptr(out_deltas), int(threads))


def orc_gauss_seidel_step(indptr, indices, weights, gt, f, frontier, out_deltas):
    args = [_c64(indptr, np.int64), _c64(indices, np.int64), _c64(weights, np.float64),
            _c64(gt, np.int8)]
    fr = _c64(frontier, np.int64)
    _load().orc_gauss_seidel_step(*[_ptr(a) for a in args], _ptr(f), _ptr(fr), len(fr),
                                  _ptr(out_deltas))


def orc_jacobi_run(indptr, indices, weights, gt, f, frontier_init, eligible, delta, max_iters,
                   threads=1):
    args = [_c64(indptr, np.int64), _c64(indices, np.int64), _c64(weights, np.float64),
            _c64(gt, np.int8)]
    fr = _c64(frontier_init, np.int64)
    n = f.shape[0]
    left = np.empty(max(n, len(fr)) + 1, dtype=np.int64)
    it, upd, warn = C.c_int64(), C.c_int64(), C.c_int64()
    mc = C.c_double()
    nl = _load().orc_jacobi_run(*[_ptr(a) for a in args], _ptr(f), n, _ptr(fr), len(fr),
                                _ptr(eligible), float(delta), int(max_iters), int(threads),
                                C.byref(it), C.byref(upd), C.byref(mc), C.byref(warn), _ptr(left))
    return it.value, upd.value, mc.value, warn.value, left[:nl].copy()


def load_reference():
    """Import the unmodified reference ``dynlp`` package (compiled reference
    in oracle/_ref, else the source tree in this container), or None."""
    if "dynlp" in sys.modules:
        return sys.modules["dynlp"]
    path = _build.reference_path()
    if path is None and os.path.isdir("/root/reference/pkg/src/dynlp"):
        path = _build.build_reference()
    if path is None:
        return None
    if path not in sys.path:
        sys.path.insert(0, path)
    os.environ.setdefault("DYNLP_KERNELS", "compiled")
    try:
        return importlib.import_module("dynlp")
    except ImportError:
        return None
