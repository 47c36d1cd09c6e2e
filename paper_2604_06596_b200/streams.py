"""Synthetic inputs for the DynLP update path (host tooling, not the hot path).

The reference produces inputs offline: ``builder.knn_graph`` /
``builder.erdos_renyi`` build a full graph and ``stream.make_stream``
(stream.py:56-183) turns it into a ``BatchUpdate`` schedule.  This module
re-implements the same *rules* for the configurations BASELINE.json names
(blobs, k-NN, 1% seeds, insert / mixed batches) so that tests and bench.py
can run without the reference:

* a vertex's stream id is its reveal position (contiguous fresh ids per
  batch, graph.py:249-252);
* an edge enters with the insert record of its later-revealed endpoint and is
  dropped if the earlier endpoint was deleted at or before that batch
  (stream.py:149-164); edges inside a batch are ordered by (owner, other);
* classes may be 0..C-1 (the reference's binary generator cannot express
  C > 2 classes).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .batch import BatchUpdate, EdgeList


@dataclass
class Blobs:
    x: np.ndarray          # (n, d) float64 features
    classes: np.ndarray    # (n,) int8 class of every point


def make_blobs(n: int, dim: int, num_classes: int, seed: int, spread: float = 10.0,
               sigma: float = 1.0, dtype=np.float64) -> Blobs:
    """Gaussian blobs: centres U(-spread, spread)^dim, isotropic sigma, labels
    uniform over the classes."""
    rng = np.random.default_rng(seed)
    centres = rng.uniform(-spread, spread, size=(num_classes, dim))
    classes = rng.integers(0, num_classes, size=n).astype(np.int8)
    x = np.empty((n, dim), dtype=dtype)
    step = 1 << 16
    for s in range(0, n, step):
        e = min(n, s + step)
        x[s:e] = centres[classes[s:e]] + sigma * rng.standard_normal((e - s, dim))
    return Blobs(x, classes)


def _symmetrize(src, dst, sim, n):
    """Union-symmetrise directed k-NN pairs, duplicates merged by max
    (builder.py:77-92, prune mode: w = cos, keep w > 0, clip to [0, 1])."""
    keep = sim > 0
    src, dst, w = src[keep], dst[keep], np.clip(sim[keep], 0.0, 1.0)
    lo = np.minimum(src, dst).astype(np.int64)
    hi = np.maximum(src, dst).astype(np.int64)
    key = lo * np.int64(n) + hi
    order = np.argsort(key, kind="stable")
    key, w = key[order], w[order]
    first = np.ones(len(key), dtype=bool)
    first[1:] = key[1:] != key[:-1]
    starts = np.flatnonzero(first)
    merged = np.maximum.reduceat(w, starts) if len(w) else w
    uk = key[starts]
    return EdgeList(uk // n, uk % n, merged.astype(np.float64))


def knn_graph_exact(x: np.ndarray, k: int, block: int = 512) -> EdgeList:
    """Cosine k-NN in fp64 with ties to the lower id (builder.py:42-92
    semantics), O(n^2) host version for test-sized inputs."""
    x = np.asarray(x, dtype=np.float64)
    n = x.shape[0]
    xn = x / np.linalg.norm(x, axis=1, keepdims=True)
    srcs, dsts, sims = [], [], []
    ids = np.arange(n)
    for s in range(0, n, block):
        e = min(n, s + block)
        sim = xn[s:e] @ xn.T
        sim[np.arange(e - s), np.arange(s, e)] = -np.inf
        order = np.lexsort((np.broadcast_to(ids, sim.shape), -sim), axis=-1)[:, :k]
        rows = np.repeat(np.arange(s, e), k)
        cols = order.ravel()
        srcs.append(rows)
        dsts.append(cols)
        sims.append(sim[rows - s, cols])
    return _symmetrize(np.concatenate(srcs), np.concatenate(dsts), np.concatenate(sims), n)


def knn_graph_torch(x: np.ndarray, k: int, device: str = "cuda", block: int = 8192) -> EdgeList:
    """Cosine k-NN for bench-scale synthetic inputs (fp32 similarity on the
    GPU).  Input-generation only: the edge set can differ from an fp64
    selection on near-ties, which does not matter for a synthetic stream."""
    import torch

    n = x.shape[0]
    xt = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(device)
    xt = torch.nn.functional.normalize(xt, dim=1)
    srcs, dsts, sims = [], [], []
    for s in range(0, n, block):
        e = min(n, s + block)
        sim = xt[s:e] @ xt.T
        sim[torch.arange(e - s, device=device), torch.arange(s, e, device=device)] = -float("inf")
        val, idx = torch.topk(sim, k, dim=1)
        srcs.append(torch.arange(s, e, device=device).repeat_interleave(k).cpu().numpy())
        dsts.append(idx.reshape(-1).cpu().numpy())
        sims.append(val.reshape(-1).double().cpu().numpy())
        del sim
    return _symmetrize(np.concatenate(srcs), np.concatenate(dsts), np.concatenate(sims), n)


def knn_graph_torch64(x: np.ndarray, k: int, device: str = "cuda", block: int = 2048) -> EdgeList:
    """Cosine k-NN in fp64 through torch (GPU GEMM + top-k), the bench's
    synthetic-stream generator.  Input generation only, shared by both bench
    arms so that the reference arm never loads this repo's CUDA library: the
    edge set equals the exact numpy selection (knn_graph_exact) except on
    sub-ulp near-ties, whose order follows the GEMM's summation order."""
    import torch

    n = x.shape[0]
    xt = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float64)).to(device)
    xt = xt / torch.linalg.vector_norm(xt, dim=1, keepdim=True)
    srcs, dsts, sims = [], [], []
    for s in range(0, n, block):
        e = min(n, s + block)
        sim = xt[s:e] @ xt.T
        sim[torch.arange(e - s, device=device), torch.arange(s, e, device=device)] = -float("inf")
        val, idx = torch.topk(sim, k, dim=1, sorted=True)
        srcs.append(np.repeat(np.arange(s, e, dtype=np.int64), k))
        dsts.append(idx.reshape(-1).cpu().numpy().astype(np.int64))
        sims.append(val.reshape(-1).cpu().numpy())
        del sim
    return _symmetrize(np.concatenate(srcs), np.concatenate(dsts), np.concatenate(sims), n)


def uniform_cube(n: int, seed: int) -> Blobs:
    """n points uniform in [0, 1]^3, class = x > 1/2 (SURVEY.md §8(d) D-2 C5:
    a single giant component with high probability at k = 10)."""
    rng = np.random.default_rng(seed)
    x = rng.random((n, 3))
    return Blobs(x, (x[:, 0] > 0.5).astype(np.int8))


def knn_graph_grid3d(x: np.ndarray, k: int, workers: int = -1) -> EdgeList:
    """Exact Euclidean k-NN of 3-D points (a k-d tree, the low-dimensional
    analogue of the grid search; ties to the lower id by stable id order),
    union-symmetrised with max-merge like builder.py:77-92.  Weight
    exp(-d^2 / 2h^2), h = the expected k-NN radius of a uniform cloud, so
    weights lie in (0, 1]."""
    from scipy.spatial import cKDTree

    n = x.shape[0]
    tree = cKDTree(x, leafsize=32, balanced_tree=False, compact_nodes=False)
    dist, idx = tree.query(x, k=k + 1, workers=workers)
    dist, idx = dist[:, 1:], idx[:, 1:]  # drop self
    h = (k / (n * 4.0 / 3.0 * np.pi)) ** (1.0 / 3.0)
    sim = np.exp(-(dist * dist) / (2.0 * h * h)).reshape(-1)
    src = np.repeat(np.arange(n, dtype=np.int64), k)
    return _symmetrize(src, idx.reshape(-1).astype(np.int64), sim, n)


def erdos_renyi_edges(n: int, avg_degree: float, seed: int, low=0.1, high=1.0) -> EdgeList:
    rng = np.random.default_rng(seed)
    m = int(rng.binomial(n * (n - 1) // 2, min(1.0, avg_degree / max(1, n - 1))))
    keys = np.empty(0, dtype=np.int64)
    while len(keys) < m:
        a = rng.integers(0, n, size=2 * (m - len(keys)) + 16)
        b = rng.integers(0, n, size=len(a))
        ok = a != b
        keys = np.unique(np.concatenate([keys, np.minimum(a, b)[ok] * n + np.maximum(a, b)[ok]]))
    keys = np.sort(rng.choice(keys, size=m, replace=False)) if len(keys) > m else keys
    w = rng.uniform(low, high, size=len(keys))
    return EdgeList(keys // n, keys % n, w)


def stratified_seeds(classes: np.ndarray, fraction: float, seed: int) -> np.ndarray:
    """Ground-truth ids: `fraction` of every class (at least one each)."""
    rng = np.random.default_rng(seed)
    out = []
    for c in np.unique(classes):
        members = np.flatnonzero(classes == c)
        take = max(1, int(round(len(members) * fraction)))
        out.append(rng.permutation(members)[:take])
    return np.sort(np.concatenate(out))


@dataclass
class Stream:
    batches: list
    source_of: np.ndarray   # stream id -> source vertex id
    classes: np.ndarray     # class of every stream id (ground truth or not)


def phased_stream(n: int, edges: EdgeList, classes: np.ndarray, gt_ids: np.ndarray,
                  batch_size: int, seed: int, insert_fraction: float = 0.99,
                  gt_fraction: float = 0.01, delete_fraction: float = 0.0,
                  initial_gt: int = 2, phases=None) -> Stream:
    """Reveal schedule with the make_stream rules (stream.py:56-183).

    ``phases`` optionally lists (num_batches, batch_size, insert_fraction,
    gt_fraction, delete_fraction) tuples run in order; the final phase
    repeats until the pools drain.  Deletes pick uniformly among alive ids.
    """
    rng = np.random.default_rng(seed)
    classes = np.asarray(classes, dtype=np.int8)
    is_gt = np.zeros(n, dtype=bool)
    is_gt[gt_ids] = True
    gt_queue = rng.permutation(np.flatnonzero(is_gt))
    unl_queue = rng.permutation(np.flatnonzero(~is_gt))
    if phases is None:
        phases = [(None, batch_size, insert_fraction, gt_fraction, delete_fraction)]
    order = [gt_queue[:initial_gt]]
    dels = [np.empty(0, dtype=np.int64)]
    gi, ui = min(initial_gt, len(gt_queue)), 0
    revealed = gi
    alive = np.zeros(n, dtype=bool)
    alive[:revealed] = True
    for count, bs, fi, fg, fd in phases:
        done = 0
        while (count is None or done < count) and (gi < len(gt_queue) or ui < len(unl_queue)):
            n_gt = int(round(fg * bs))
            n_del = int(round(fd * bs))
            n_unl = bs - n_gt - n_del
            left_gt, left_unl = len(gt_queue) - gi, len(unl_queue) - ui
            take_gt, take_unl = min(n_gt, left_gt), min(n_unl, left_unl)
            short = n_gt + n_unl - take_gt - take_unl  # refill from the other pool
            extra = min(short, left_unl - take_unl)
            take_unl += extra
            take_gt += min(short - extra, left_gt - take_gt)
            if take_gt + take_unl == 0:
                break
            alive_ids = np.flatnonzero(alive[:revealed])
            nd = min(n_del, max(0, len(alive_ids) - 1))
            d = np.sort(rng.choice(alive_ids, size=nd, replace=False)) if nd else np.empty(0, np.int64)
            alive[d] = False
            ins = np.concatenate([unl_queue[ui:ui + take_unl], gt_queue[gi:gi + take_gt]])
            ui += take_unl
            gi += take_gt
            order.append(ins)
            dels.append(d.astype(np.int64))
            alive[revealed:revealed + len(ins)] = True
            revealed += len(ins)
            done += 1
    source_of = np.concatenate(order).astype(np.int64)
    stream_of = np.full(n, -1, dtype=np.int64)
    stream_of[source_of] = np.arange(len(source_of))
    bounds = np.cumsum([0] + [len(o) for o in order])
    nb = len(order)
    reveal_batch = np.searchsorted(bounds[1:], np.arange(revealed), side="right")
    death_batch = np.full(revealed, nb + 1, dtype=np.int64)
    for t, d in enumerate(dels):
        death_batch[d] = t
    sa, sb = stream_of[edges.u], stream_of[edges.v]
    ok = (sa >= 0) & (sb >= 0)
    sa, sb, ew = sa[ok], sb[ok], edges.w[ok]
    owner, other = np.maximum(sa, sb), np.minimum(sa, sb)
    keep = death_batch[other] > reveal_batch[owner]
    owner, other, ew = owner[keep], other[keep], ew[keep]
    o = np.lexsort((other, owner))
    owner, other, ew = owner[o], other[o], ew[o]
    eb = np.searchsorted(bounds[1:], owner, side="right")
    ebounds = np.searchsorted(eb, np.arange(nb + 1))
    stream_classes = classes[source_of]
    batches = []
    for t in range(nb):
        lo, hi = bounds[t], bounds[t + 1]
        g = np.where(is_gt[source_of[lo:hi]], stream_classes[lo:hi], -1).astype(np.int8)
        el, eh = ebounds[t], ebounds[t + 1]
        batches.append(BatchUpdate(
            t=t, insert_ids=np.arange(lo, hi, dtype=np.int64), insert_gt=g,
            edge_owner=(owner[el:eh] - lo).astype(np.int64), edge_other=other[el:eh].astype(np.int64),
            edge_w=ew[el:eh].astype(np.float64), deletes=dels[t]))
    return Stream(batches, source_of, stream_classes)


def single_batch(n: int, edges: EdgeList, gt: dict | None = None) -> BatchUpdate:
    """Whole graph as one batch with ids kept (stream.py:186-208 rules)."""
    g = np.full(n, -1, dtype=np.int8)
    for v, c in (gt or {}).items():
        g[int(v)] = int(c)
    owner = np.maximum(edges.u, edges.v)
    other = np.minimum(edges.u, edges.v)
    o = np.lexsort((other, owner))
    return BatchUpdate(t=0, insert_ids=np.arange(n, dtype=np.int64), insert_gt=g,
                       edge_owner=owner[o].astype(np.int64), edge_other=other[o].astype(np.int64),
                       edge_w=np.asarray(edges.w, dtype=np.float64)[o],
                       deletes=np.empty(0, dtype=np.int64))


def merge_batches(batches) -> BatchUpdate:
    """Concatenate consecutive pure-insert batches into one bootstrap batch."""
    ids, gts, own, oth, ws = [], [], [], [], []
    off = 0
    for b in batches:
        if len(b.deletes):
            raise ValueError("merge_batches only merges insert-only batches")
        ids.append(b.insert_ids)
        gts.append(b.insert_gt)
        own.append(b.edge_owner + off)
        oth.append(b.edge_other)
        ws.append(b.edge_w)
        off += len(b.insert_ids)
    return BatchUpdate(t=batches[-1].t, insert_ids=np.concatenate(ids), insert_gt=np.concatenate(gts),
                       edge_owner=np.concatenate(own), edge_other=np.concatenate(oth),
                       edge_w=np.concatenate(ws), deletes=np.empty(0, dtype=np.int64))
