"""Drop-in for the reference's k-NN graph builder on the B200.

Mirrors ``FeatureMatrix`` / ``knn_graph`` of
/root/reference/pkg/src/dynlp/builder.py:18-92 (same arguments, validation
messages and EdgeList output sorted by (lo, hi)), plus ``knn_query`` -- the
k-NN rows of a batch of arriving points against the whole dataset, i.e. the
per-batch edge construction of a stream.  Execution: tensor-core screen
(tcgen05, fp16 hi/lo split, fp32 accumulation in TMEM) + exact fp64
re-check with a certificate (csrc/knn.cu); there is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _native
from .batch import EdgeList
from .errors import CudaError, ValidationError

SIMILARITY_PRUNE = "prune"
SIMILARITY_AFFINE = "affine"


@dataclass
class FeatureMatrix:
    """Dense per-item feature vectors (builder.py:18-39)."""

    rows: np.ndarray
    item_ids: Optional[np.ndarray] = None
    true_labels: Optional[np.ndarray] = None

    def __post_init__(self) -> None:
        self.rows = np.ascontiguousarray(self.rows, dtype=np.float64)
        if self.rows.ndim != 2:
            raise ValidationError("feature matrix must be 2-D")
        if self.item_ids is None:
            self.item_ids = np.arange(self.rows.shape[0], dtype=np.int64)

    @property
    def n(self) -> int:
        return self.rows.shape[0]


@dataclass
class KnnStats:
    screen_ms: float
    recheck_ms: float
    exact_ms: float
    fallback_queries: int
    queries: int
    eps: float


class KnnIndex:
    """Device-resident normalised features + tensor-core operands."""

    def __init__(self, features, device: int = 0) -> None:
        self._lib = _native.load()
        h = C.c_void_p()
        rc = self._lib.dlp_knn_create(int(device), C.byref(h))
        if rc != 0 or not h.value:
            raise CudaError(f"dlp_knn_create failed on device {device} (rc={rc}); a B200 (sm_100a) is required")
        self._h = h
        fm = features if isinstance(features, FeatureMatrix) else FeatureMatrix(features)
        self.n = fm.n
        self._check(self._lib.dlp_knn_set_features(self._h, fm.rows.ctypes.data, fm.rows.shape[0],
                                                   fm.rows.shape[1]))

    def _check(self, rc):
        if rc == 0:
            return
        msg = self._lib.dlp_knn_last_error(self._h).decode()
        if rc == 3:
            raise ValidationError(msg)
        raise CudaError(msg)

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._lib.dlp_knn_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def query(self, q0: int, q1: int, k: int):
        """(ids, sims) of shape (q1-q0, k): rows ordered by (-sim, id)."""
        nq = int(q1) - int(q0)
        ids = np.empty((max(nq, 0), k), dtype=np.int64)
        sims = np.empty((max(nq, 0), k), dtype=np.float64)
        self._check(self._lib.dlp_knn_query(self._h, int(q0), int(q1), int(k), ids.ctypes.data,
                                            sims.ctypes.data))
        return ids, sims

    def graph(self, k: int, similarity_mode: str = SIMILARITY_PRUNE) -> EdgeList:
        if similarity_mode not in (SIMILARITY_PRUNE, SIMILARITY_AFFINE):
            raise ValidationError(f"unknown similarity mode {similarity_mode!r}")
        m = C.c_int64()
        self._check(self._lib.dlp_knn_graph(self._h, int(k), 1 if similarity_mode == SIMILARITY_AFFINE else 0,
                                            C.byref(m)))
        u = np.empty(m.value, dtype=np.int64)
        v = np.empty(m.value, dtype=np.int64)
        w = np.empty(m.value, dtype=np.float64)
        self._check(self._lib.dlp_knn_read_edges(self._h, u.ctypes.data, v.ctypes.data, w.ctypes.data, m.value))
        return EdgeList(u, v, w)

    def stats(self) -> KnnStats:
        a, b, c, e = C.c_double(), C.c_double(), C.c_double(), C.c_double()
        nf, nq = C.c_int64(), C.c_int64()
        self._check(self._lib.dlp_knn_stats(self._h, C.byref(a), C.byref(b), C.byref(c), C.byref(nf), C.byref(nq),
                                            C.byref(e)))
        return KnnStats(a.value, b.value, c.value, nf.value, nq.value, e.value)

    KP = 16  # candidates per list (csrc/knn.cu)

    def debug_candidates(self, q0: int, q1: int):
        """Screened candidates of the last query call: (lists, val, id, thr)."""
        nq = q1 - q0
        cap = nq * 64 * self.KP
        ns = C.c_int32()
        val = np.empty(cap, dtype=np.float32)
        ids = np.empty(cap, dtype=np.int32)
        thr = np.empty(nq * 64, dtype=np.float32)
        self._check(self._lib.dlp_knn_debug_candidates(self._h, q0, q1, C.byref(ns), val.ctypes.data,
                                                       ids.ctypes.data, thr.ctypes.data, cap))
        s, kp = ns.value, self.KP
        return s, val[:nq * s * kp].reshape(nq, s * kp), ids[:nq * s * kp].reshape(nq, s * kp), \
            thr[:nq * s].reshape(nq, s)


def knn_graph(features, k: int, similarity_mode: str = SIMILARITY_PRUNE, block: int = 512,
              device: int = 0) -> EdgeList:
    """builder.knn_graph: union-symmetrised cosine k-NN graph, ties toward the
    lower id, duplicate directed edges merged by max, weights = cos (prune,
    non-positive dropped) or (1+cos)/2 (affine).  `block` is accepted for
    signature parity (the GPU tiles the problem itself)."""
    fm = features if isinstance(features, FeatureMatrix) else FeatureMatrix(features)
    n = fm.n
    if not 1 <= k < n:
        raise ValidationError(f"k must be in [1, {n - 1}]")
    if similarity_mode not in (SIMILARITY_PRUNE, SIMILARITY_AFFINE):
        raise ValidationError(f"unknown similarity mode {similarity_mode!r}")
    idx = KnnIndex(fm, device)
    try:
        return idx.graph(k, similarity_mode)
    finally:
        idx.close()
