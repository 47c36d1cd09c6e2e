"""CPU restatement of the reference k-NN graph builder (TEST INFRASTRUCTURE ONLY).

Follows /root/reference/pkg/src/dynlp/builder.py step by step:
  :30-33  all-zero rows rejected
  :54-57  k in [1, n-1], mode in {prune, affine}
  :59     x / ||x|| in fp64 (np.linalg.norm, axis=1)
  :62-65  block sims x[a:b] @ x.T, self = -inf
  :66-68  order by (-sim, id), first k
  :74-82  w = cos or (1+cos)/2, keep w > 0, clip [0, 1]
  :85-92  lo/hi keys, np.unique, max-merge
Pinned against tests/golden/knn_reference.npz (the real reference's output).
Only tests/ may import this module.
"""

from __future__ import annotations

import numpy as np


class OracleValidationError(ValueError):
    pass


def knn_topk(x: np.ndarray, k: int, block: int = 512):
    """Directed top-k rows: ids (n, k) and sims (n, k)."""
    x = np.asarray(x, dtype=np.float64)
    norms = np.linalg.norm(x, axis=1)
    zero = np.flatnonzero(norms == 0)
    if len(zero):
        raise OracleValidationError(f"all-zero feature row {int(zero[0])} (cosine undefined)")
    n = x.shape[0]
    if not 1 <= k < n:
        raise OracleValidationError(f"k must be in [1, {n - 1}]")
    xn = x / norms[:, None]
    ids = np.empty((n, k), dtype=np.int64)
    sims = np.empty((n, k), dtype=np.float64)
    all_ids = np.arange(n)
    for a in range(0, n, block):
        b = min(a + block, n)
        s = xn[a:b] @ xn.T
        s[np.arange(b - a), np.arange(a, b)] = -np.inf
        order = np.lexsort((np.broadcast_to(all_ids, s.shape), -s), axis=-1)[:, :k]
        ids[a:b] = order
        sims[a:b] = np.take_along_axis(s, order, axis=1)
    return ids, sims


def knn_graph(x: np.ndarray, k: int, mode: str = "prune", block: int = 512):
    if mode not in ("prune", "affine"):
        raise OracleValidationError(f"unknown similarity mode {mode!r}")
    ids, sims = knn_topk(x, k, block)
    n = ids.shape[0]
    src = np.repeat(np.arange(n), k)
    dst = ids.ravel()
    sim = sims.ravel()
    w = (1.0 + sim) / 2.0 if mode == "affine" else sim
    keep = w > 0
    src, dst, w = src[keep], dst[keep], np.clip(w[keep], 0.0, 1.0)
    if len(src) == 0:
        return np.empty(0, np.int64), np.empty(0, np.int64), np.empty(0, np.float64)
    lo, hi = np.minimum(src, dst), np.maximum(src, dst)
    key = lo.astype(np.int64) * n + hi
    uniq, inv = np.unique(key, return_inverse=True)
    merged = np.full(len(uniq), -np.inf)
    np.maximum.at(merged, inv, w)
    return (uniq // n).astype(np.int64), (uniq % n).astype(np.int64), merged
