"""Drop-in host API for the DynLP batch update, executed on a B200.

Mirrors the reference's engine surface (/root/reference/pkg/src/dynlp/):

* ``EngineConfig``      engine.py:40-70   (same fields, same validation)
* ``IterationReport``   engine.py:104-129 (+ edges_traversed, certify_sweeps)
* ``DynamicGraph``      graph.py:176      -- here a handle on the device engine
                                            that owns graph AND labels in HBM
* ``LabelState``        labels.py:13      -- a view of the labels held on device
* ``apply_batch``       engine.py:328-413
* ``apply_batch_structure`` engine.py:141-156
* ``run_batches``       engine.py:416-423
* ``itlp_batch_solve``  baselines.py:236-253
* ``harmonic_solve`` / ``oracle_batch_solve`` / ``stlp_batch_solve``
                        baselines.py:163-190, 321-371 (dense Cholesky on the
                        device, cuSOLVER)

Everything below the C-ABI (include/dynlp_b200.h) runs as sm_100a CUDA
kernels; this module only marshals arguments and maps status codes onto the
reference's exception types.
"""

from __future__ import annotations

import ctypes as C
import math
import os
import time
from dataclasses import dataclass, field
from typing import Optional, Union

import numpy as np

from . import _native
from .batch import BatchUpdate, EdgeList, as_arrays
from .errors import CudaError, FileFormatError, InternalError, ValidationError

MODE_JACOBI = "parallel_jacobi"
MODE_GAUSS_SEIDEL = "sequential_gauss_seidel"
DEFAULT_DELTA = 1e-4
MAX_ITERATIONS_PER_VERTEX = 10
UNLABELED = -1
DENSE_SOLVE_CAP = 5000  # baselines.py:29


@dataclass
class EngineConfig:
    delta: float = DEFAULT_DELTA
    tau: Union[float, str] = "auto"
    max_iterations: Optional[int] = None  # None: 10x the alive vertex count
    mode: str = MODE_JACOBI
    threads: Optional[int] = None  # accepted for signature parity; unused on the GPU
    component_init: bool = True

    def validate(self) -> None:
        if not self.delta > 0:
            raise ValidationError("delta must be positive")
        if self.max_iterations is not None and self.max_iterations < 1:
            raise ValidationError("max_iterations must be >= 1")
        if self.mode not in (MODE_JACOBI, MODE_GAUSS_SEIDEL):
            raise ValidationError(f"unknown mode {self.mode!r}")
        if isinstance(self.tau, str):
            if self.tau != "auto":
                raise ValidationError("tau must be a number or 'auto'")
        elif self.tau < 0:
            raise ValidationError("tau must be nonnegative")

    def resolved_threads(self) -> int:
        return max(1, int(self.threads)) if self.threads is not None else (os.cpu_count() or 1)

    def resolved_max_iterations(self, num_alive: int) -> int:
        if self.max_iterations is not None:
            return self.max_iterations
        return max(1, MAX_ITERATIONS_PER_VERTEX * num_alive)

    def _c(self, num_classes: int) -> _native.Config:
        return _native.Config(
            float(self.delta), math.nan if self.tau == "auto" else float(self.tau),
            0 if self.max_iterations is None else int(self.max_iterations),
            1 if self.component_init else 0, 0 if self.mode == MODE_JACOBI else 1,
            int(num_classes), 0)


@dataclass
class IterationReport:
    method: str = "dynlp"
    t: int = 0
    iterations: int = 0
    updates: int = 0
    max_change: float = 0.0
    converged: bool = True
    warnings: int = 0
    isolated_pinned: int = 0
    unreachable_pinned: int = 0
    wall_time_ms: float = 0.0
    edges_traversed: int = 0
    certify_sweeps: int = 0
    lp_kernel_ms: float = 0.0
    gpu_launches: int = 0
    lp_rounds: int = 0
    lp_union_rows: int = 0
    lp_union_entries: int = 0

    def to_json_dict(self) -> dict:
        return {k: getattr(self, k) for k in (
            "method", "t", "iterations", "updates", "max_change", "converged", "warnings",
            "isolated_pinned", "unreachable_pinned", "wall_time_ms")}


@dataclass
class CsrView:
    indptr: np.ndarray
    indices: np.ndarray
    weights: np.ndarray
    degrees: np.ndarray


def _raise(lib, h, rc, where="dynlp"):
    msg = lib.dlp_last_error(h).decode() if h else "engine creation failed"
    if rc == 3:
        raise ValidationError(msg)
    if rc == 4:
        raise FileFormatError(msg)
    if rc == 5:
        raise CudaError(f"{where}: {msg}")
    raise InternalError(f"{where}: {msg}")


class DynamicGraph:
    """Device-resident DynLP state on one GPU: graph (adjacency rows, edge
    log, components) and labels (one fp64 column per class, one column for
    binary).  Created empty, like the reference's ``DynamicGraph()``."""

    def __init__(self, device: int = 0, num_classes: int = 2) -> None:
        self._lib = _native.load()
        self.device = int(device)
        self.num_classes = max(2, int(num_classes))
        cfg = EngineConfig()._c(self.num_classes)
        h = C.c_void_p()
        rc = self._lib.dlp_create(C.byref(cfg), self.device, C.byref(h))
        if rc == 3:
            raise ValidationError(f"num_classes must be <= 16 (got {self.num_classes})")
        if rc != 0 or not h.value:
            raise CudaError(f"dlp_create failed on device {device} (rc={rc}); a B200 (sm_100a) is required")
        self._h = h
        self.ncol = int(self._lib.dlp_num_columns(self._h))
        self._version = 0

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._lib.dlp_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def reserve(self, n_vertices: int, n_edges: int) -> None:
        """Capacity hint: pre-size device arrays for n_vertices slots and
        n_edges live edges (no reallocation inside later batches)."""
        self._check(self._lib.dlp_reserve(self._h, int(n_vertices), int(n_edges)))

    # -- accessors mirroring graph.py ------------------------------------------------
    def _counts(self):
        n, a = C.c_int64(), C.c_int64()
        self._lib.dlp_num_slots(self._h, C.byref(n), C.byref(a))
        return n.value, a.value

    @property
    def num_slots(self) -> int:
        return self._counts()[0]

    @property
    def num_alive(self) -> int:
        return self._counts()[1]

    def _stats(self):
        m, tau = C.c_int64(), C.c_double()
        self._lib.dlp_graph_stats(self._h, C.byref(m), C.byref(tau))
        return m.value, tau.value

    @property
    def edge_count(self) -> int:
        return self._stats()[0]

    @property
    def last_tau(self) -> float:
        return self._stats()[1]

    @property
    def alive(self) -> np.ndarray:
        n = self.num_slots
        a = np.empty(n, dtype=np.uint8)
        self._check(self._lib.dlp_read_alive(self._h, _native.ptr(a), n))
        return a.astype(bool)

    def alive_ids(self) -> np.ndarray:
        return np.flatnonzero(self.alive).astype(np.int64)

    def is_alive(self, u: int) -> bool:
        return 0 <= u < self.num_slots and bool(self.alive[u])

    def csr(self) -> CsrView:
        n = self.num_slots
        m = self.edge_count
        indptr = np.empty(n + 1, dtype=np.int64)
        indices = np.empty(2 * m, dtype=np.int64)
        weights = np.empty(2 * m, dtype=np.float64)
        degrees = np.empty(n, dtype=np.float64)
        self._check(self._lib.dlp_read_csr(self._h, _native.ptr(indptr), _native.ptr(indices),
                                           _native.ptr(weights), _native.ptr(degrees), n, 2 * m))
        return CsrView(indptr, indices, weights, degrees)

    def live_edges(self) -> EdgeList:
        m = self.edge_count
        u = np.empty(m, dtype=np.int64)
        v = np.empty(m, dtype=np.int64)
        w = np.empty(m, dtype=np.float64)
        self._check(self._lib.dlp_read_live_edges(self._h, _native.ptr(u), _native.ptr(v),
                                                  _native.ptr(w), m))
        return EdgeList(u, v, w)

    def neighbors(self, u: int):
        if not self.is_alive(u):
            raise ValidationError(f"vertex {u} is deleted" if 0 <= u < self.num_slots
                                  else f"unknown vertex id {u}")
        c = self.csr()
        return c.indices[c.indptr[u]:c.indptr[u + 1]], c.weights[c.indptr[u]:c.indptr[u + 1]]

    def weighted_degree(self, u: int) -> float:
        return float(self.neighbors(u)[1].sum())

    def eligible(self) -> np.ndarray:
        n = self.num_slots
        a = np.empty(n, dtype=np.uint8)
        self._check(self._lib.dlp_read_eligible(self._h, _native.ptr(a), n))
        return a.astype(bool)

    def intra_labeling(self):
        """(vertices, parent, component_id) of the last batch's find_components."""
        cap = self.num_slots + 1
        v = np.empty(cap, np.int64)
        p = np.empty(cap, np.int64)
        c = np.empty(cap, np.int64)
        k = C.c_int64()
        self._check(self._lib.dlp_read_intra(self._h, _native.ptr(v), _native.ptr(p),
                                             _native.ptr(c), cap, C.byref(k)))
        return v[:k.value], p[:k.value], c[:k.value]

    def allocate_ids(self, k: int) -> np.ndarray:
        n = self.num_slots
        return np.arange(n, n + k, dtype=np.int64)

    # -- labels ---------------------------------------------------------------------
    def read_labels(self):
        n = self.num_slots
        f = np.empty((self.ncol, n), dtype=np.float64)
        gt = np.empty(n, dtype=np.int8)
        self._check(self._lib.dlp_read_labels(self._h, _native.ptr(f), _native.ptr(gt), n))
        return f, gt

    def write_labels(self, f) -> None:
        n = self.num_slots
        f = np.ascontiguousarray(f, dtype=np.float64).reshape(self.ncol, n)
        self._check(self._lib.dlp_write_labels(self._h, _native.ptr(f), n))
        self._version += 1

    def harmonic(self, stlp: bool = False, dense_cap: int = DENSE_SOLVE_CAP):
        """Closed-form harmonic labels on the device: (C, n) array and the
        count of alive vertices pinned to 0.5 as unreachable."""
        n = self.num_slots
        f = np.empty((self.ncol, n), dtype=np.float64)
        unr = np.zeros(1, dtype=np.int64)
        self._check(self._lib.dlp_harmonic_solve(self._h, int(bool(stlp)), int(dense_cap), _native.ptr(f), n,
                                                 _native.ptr(unr)))
        return f, int(unr[0])

    def _check(self, rc):
        if rc != 0:
            _raise(self._lib, self._h, rc)

    # -- batch application ------------------------------------------------------------
    def _run_arrays(self, fn_name, arrays, cfg: Optional[EngineConfig]):
        t, ids, gt, owner, other, w, dels = arrays
        b = _native.Batch(t, len(ids), _native.ptr(ids), _native.ptr(gt), len(owner),
                          _native.ptr(owner), _native.ptr(other), _native.ptr(w), len(dels),
                          _native.ptr(dels))
        fn = getattr(self._lib, fn_name)
        if cfg is None:
            rc = fn(self._h, C.byref(b))
            reps = None
        else:
            reps = (_native.Report * self.ncol)()
            c = cfg._c(self.num_classes)
            rc = fn(self._h, C.byref(c), C.byref(b), reps)
        self._version += 1
        if rc != 0:
            _raise(self._lib, self._h, rc)
        return reps

    def _run_pipelined(self, batch, next_batch, cfg: EngineConfig):
        # the arrays of both batches must outlive the call; keep the staged
        # batch's arrays referenced until the next call consumes them
        cur = as_arrays(batch) if getattr(self, "_staged_src", (None,))[0] is not batch else self._staged_arrays
        nxt = as_arrays(next_batch)
        t, ids, gt, owner, other, w, dels = cur
        b = _native.Batch(t, len(ids), _native.ptr(ids), _native.ptr(gt), len(owner), _native.ptr(owner),
                          _native.ptr(other), _native.ptr(w), len(dels), _native.ptr(dels))
        t2, ids2, gt2, owner2, other2, w2, dels2 = nxt
        b2 = _native.Batch(t2, len(ids2), _native.ptr(ids2), _native.ptr(gt2), len(owner2), _native.ptr(owner2),
                           _native.ptr(other2), _native.ptr(w2), len(dels2), _native.ptr(dels2))
        reps = (_native.Report * self.ncol)()
        c = cfg._c(self.num_classes)
        rc = self._lib.dlp_apply_batch_pipelined(self._h, C.byref(c), C.byref(b), C.byref(b2), reps)
        self._staged_src, self._staged_arrays = (next_batch,), nxt
        self._version += 1
        if rc != 0:
            _raise(self._lib, self._h, rc)
        return reps

    def _run(self, fn_name, batch, cfg: Optional[EngineConfig]):
        if getattr(self, "_staged_src", (None,))[0] is batch:
            batch_arrays = self._staged_arrays  # same buffers the engine staged
            self._staged_src = (None,)
            return self._run_arrays(fn_name, batch_arrays, cfg)
        return self._run_arrays(fn_name, as_arrays(batch), cfg)

    def apply_device(self, dev_batch: dict, cfg: EngineConfig, trusted: bool = True):
        """apply_batch with batch arrays already in device memory (torch
        tensors or raw pointers): the bench's HBM-resident leg."""
        def p(x):
            return x if isinstance(x, int) else (x.data_ptr() if x is not None else None)
        b = _native.Batch(int(dev_batch.get("t", 0)), int(dev_batch["n_ins"]),
                          p(dev_batch["insert_ids"]), p(dev_batch["insert_gt"]),
                          int(dev_batch["n_edges"]), p(dev_batch["edge_owner"]),
                          p(dev_batch["edge_other"]), p(dev_batch["edge_w"]),
                          int(dev_batch["n_del"]), p(dev_batch["deletes"]))
        reps = (_native.Report * self.ncol)()
        c = cfg._c(self.num_classes)
        rc = self._lib.dlp_apply_batch_device(self._h, C.byref(c), C.byref(b), 1 if trusted else 0, reps)
        self._version += 1
        if rc != 0:
            _raise(self._lib, self._h, rc)
        return _reports(reps, "dynlp")


def _reports(reps, method):
    return [IterationReport(method=method, t=r.t, iterations=r.iterations, updates=r.updates,
                            max_change=r.max_change, converged=bool(r.converged),
                            warnings=r.warnings, isolated_pinned=r.isolated_pinned,
                            unreachable_pinned=r.unreachable_pinned,
                            wall_time_ms=r.wall_time_ms, edges_traversed=r.edges_traversed,
                            certify_sweeps=r.certify_sweeps, lp_kernel_ms=r.lp_kernel_ms,
                            gpu_launches=r.gpu_launches, lp_rounds=r.lp_rounds,
                            lp_union_rows=r.lp_union_rows, lp_union_entries=r.lp_union_entries)
            for r in reps]


class LabelState:
    """Fractional labels and ground truth (labels.py:13-64), held on device.

    ``f`` is the binary label vector (column 0) and ``F`` the (C, n) matrix
    of one-vs-rest columns; both are read from HBM on access (cached until the
    next batch).  ``gt`` is the raw class per slot (-1 unlabeled)."""

    def __init__(self, n: int = 0) -> None:
        self._graph: Optional[DynamicGraph] = None
        self._cache = None
        self._cache_version = -1

    def _bind(self, graph: DynamicGraph) -> None:
        if self._graph is not None and self._graph is not graph:
            raise ValidationError("LabelState is bound to a different graph")
        self._graph = graph

    def _load(self):
        g = self._graph
        if g is None:
            return np.empty((1, 0)), np.empty(0, np.int8)
        if self._cache_version != g._version:
            self._cache = g.read_labels()
            self._cache_version = g._version
        return self._cache

    @property
    def F(self) -> np.ndarray:
        return self._load()[0]

    @property
    def f(self) -> np.ndarray:
        return self._load()[0][0]

    @property
    def gt(self) -> np.ndarray:
        return self._load()[1]

    @property
    def n(self) -> int:
        return self._load()[1].shape[0]

    def argmax(self) -> np.ndarray:
        """Class per vertex: binary_label for C=2, else the column argmax
        (ties to the lowest class index)."""
        F = self.F
        if F.shape[0] == 1:
            return (F[0] >= 0.5).astype(np.int8)
        return np.argmax(F, axis=0).astype(np.int8)

    def class_ids(self, graph: DynamicGraph, cls: int) -> np.ndarray:
        return np.flatnonzero(graph.alive & (self.gt[: graph.num_slots] == cls)).astype(np.int64)

    def unlabeled_ids(self, graph: DynamicGraph) -> np.ndarray:
        return np.flatnonzero(graph.alive & (self.gt[: graph.num_slots] == UNLABELED)).astype(np.int64)


def binary_label(value: float) -> int:
    """labels.py:67-69: ties go to class 1."""
    return 1 if value >= 0.5 else 0


def _result(graph, reports):
    return reports[0] if graph.ncol == 1 else reports


def apply_batch(graph: DynamicGraph, labels: LabelState, batch, cfg: EngineConfig, next_batch=None):
    """engine.apply_batch: returns (labels, IterationReport) for binary runs,
    (labels, [IterationReport per class column]) for C > 2.

    ``next_batch`` (optional, B200 ingestion pipeline): the batch the caller
    will apply next; it is validated and copied to the device while this
    batch's kernels run, and the next call with the same object skips both
    steps.  Results are identical either way."""
    cfg.validate()
    labels._bind(graph)
    if next_batch is None:
        reps = graph._run("dlp_apply_batch", batch, cfg)
    else:
        reps = graph._run_pipelined(batch, next_batch, cfg)
    return labels, _result(graph, _reports(reps, "dynlp"))


def apply_batch_structure(graph: DynamicGraph, labels: LabelState, batch) -> None:
    labels._bind(graph)
    graph._run("dlp_apply_structure", batch, None)


def run_batches(graph: DynamicGraph, labels: LabelState, batches, cfg: EngineConfig, pipelined: bool = True):
    """engine.run_batches; with ``pipelined`` each batch's validation and
    host-to-device copy overlap the previous batch's propagation."""
    batches = list(batches)
    out = []
    for i, b in enumerate(batches):
        nxt = batches[i + 1] if pipelined and i + 1 < len(batches) else None
        out.append(apply_batch(graph, labels, b, cfg, next_batch=nxt)[1])
    return out


def harmonic_solve(graph: DynamicGraph, labels: LabelState, dense_cap: int = DENSE_SOLVE_CAP,
                   return_info: bool = False):
    """baselines.harmonic_solve (baselines.py:163-190) on the device: the
    closed-form labels of the current graph, unreachable vertices at 0.5.
    Binary engines return the (n,) vector, C-column engines (C, n)."""
    labels._bind(graph)
    f, unr = graph.harmonic(False, dense_cap)
    out = f[0] if graph.ncol == 1 else f
    return (out, {"unreachable_pinned": unr}) if return_info else out


def _solve_batch(graph, labels, batch, stlp, dense_cap, method):
    started = time.perf_counter()
    apply_batch_structure(graph, labels, batch)
    f, _ = graph.harmonic(stlp, dense_cap)
    gt = labels.gt
    unl = np.flatnonzero(graph.alive & (gt[: graph.num_slots] == UNLABELED))
    cur = labels.F.copy()
    cur[:, unl] = f[:, unl]
    graph.write_labels(cur)
    reps = []
    for _ in range(graph.ncol):
        r = IterationReport(method=method, t=int(batch.t), iterations=1, updates=len(unl), converged=True)
        r.wall_time_ms = (time.perf_counter() - started) * 1000.0
        reps.append(r)
    return labels, _result(graph, reps)


def oracle_batch_solve(graph: DynamicGraph, labels: LabelState, batch, cfg: EngineConfig,
                       dense_cap: int = DENSE_SOLVE_CAP):
    """baselines.oracle_batch_solve (baselines.py:346-371): structure, then the
    closed-form solution of the whole graph."""
    return _solve_batch(graph, labels, batch, False, dense_cap, "oracle")


def stlp_batch_solve(graph: DynamicGraph, labels: LabelState, batch, cfg: EngineConfig,
                     dense_cap: int = DENSE_SOLVE_CAP):
    """baselines.stlp_batch_solve (baselines.py:321-343): structure, then the
    short-circuit solve (same linear system; both classes must be present)."""
    return _solve_batch(graph, labels, batch, True, dense_cap, "stlp")


def itlp_batch_solve(graph: DynamicGraph, labels: LabelState, batch, cfg: EngineConfig):
    """baselines.itlp_batch_solve: structure, then full sweeps to delta."""
    cfg.validate()
    labels._bind(graph)
    reps = graph._run("dlp_itlp_batch", batch, cfg)
    return labels, _result(graph, _reports(reps, "itlp"))
