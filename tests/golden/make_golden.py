"""Generate tests/golden/*.npz by running the REAL reference (this container only).

    python tests/golden/make_golden.py

Imports the unmodified reference ``dynlp`` (compiled backend, via
oracle.load_reference(): the Cython build in oracle/_ref or the source tree
under /root/reference) and records, for several batch streams, every
output the DynLP update path defines:

* per batch: f (all slots, every label column), the IterationReport fields,
  tau (resolve_tau, engine.py:182-188), the eligible mask (alive & unlabeled
  & reachable, engine.py:350-361), the intra-batch labeling
  (components.py:84-124) and a SHA-256 of the CSR snapshot
  (graph.py:218-231);
* the final CSR in full.

For C > 2 classes the reference is binary-only (labels.py:42-43), so each
column c is an independent reference run with ground truth remapped to
1 for class c and 0 for the other classes.

Kernel-level fixtures record jacobi_step / jacobi_run of the compiled
``_csr`` on random CSR states (tests/test_kernels.py:14-20 style) plus the
degenerate cases the reference tests pin (isolated sentinel, zero weights,
duplicate frontier entries).
"""

from __future__ import annotations

import copy
import hashlib
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import load_reference  # noqa: E402
from paper_2604_06596_b200 import streams  # noqa: E402
from paper_2604_06596_b200.batch import BatchUpdate as OwnBatch  # noqa: E402

ref = load_reference()
assert ref is not None, "reference not importable"
import dynlp.kernels as rk  # noqa: E402

assert rk.BACKEND == "compiled", rk.BACKEND
from dynlp.components import IntraBatchGraph, find_components  # noqa: E402
from dynlp.engine import EngineConfig, apply_batch, reachable_mask, resolve_tau  # noqa: E402
from dynlp.graph import BatchUpdate, DynamicGraph, EdgeList  # noqa: E402
from dynlp.labels import LabelState  # noqa: E402


def to_ref(b) -> BatchUpdate:
    return BatchUpdate(t=int(b.t), insert_ids=np.asarray(b.insert_ids, np.int64),
                       insert_gt=np.asarray(b.insert_gt, np.int8),
                       edge_owner=np.asarray(b.edge_owner, np.int64),
                       edge_other=np.asarray(b.edge_other, np.int64),
                       edge_w=np.asarray(b.edge_w, np.float64),
                       deletes=np.asarray(b.deletes, np.int64))


def remap(b, c):
    out = copy.copy(b)
    g = np.asarray(b.insert_gt)
    out.insert_gt = np.where(g < 0, -1, np.where(g == c, 1, 0)).astype(np.int8)
    return out


def csr_digest(graph):
    csr = graph.csr()
    h = hashlib.sha256()
    for a in (csr.indptr.astype(np.int64), csr.indices.astype(np.int64),
              csr.weights.astype(np.float64), csr.degrees.astype(np.float64)):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def run_case(name, batches, num_classes=2, delta=1e-6, tau="auto", max_iterations=None,
             component_init=True, mode="parallel_jacobi"):
    ncol = 1 if num_classes <= 2 else num_classes
    cfg = EngineConfig(delta=delta, tau=tau, max_iterations=max_iterations,
                       component_init=component_init, mode=mode, threads=1)
    nb = len(batches)
    f_cols = [[] for _ in range(ncol)]
    rep_i = np.zeros((nb, ncol, 6), dtype=np.int64)
    rep_mc = np.zeros((nb, ncol), dtype=np.float64)
    taus, eligs, digests, intra, slots = [], [], [], [], []
    final = None
    for c in range(ncol):
        graph, labels = DynamicGraph(), LabelState()
        for t, b in enumerate(batches):
            rb = to_ref(b if ncol == 1 else remap(b, c))
            labels, r = apply_batch(graph, labels, rb, cfg)
            rep_i[t, c] = [r.iterations, r.updates, int(r.converged), r.warnings,
                           r.isolated_pinned, r.unreachable_pinned]
            rep_mc[t, c] = r.max_change
            f_cols[c].append(labels.f[: graph.num_slots].copy())
            if c == 0:
                n = graph.num_slots
                slots.append(n)
                tv = resolve_tau(graph, cfg)
                taus.append(tv)
                elig = graph.alive & (labels.gt[:n] == -1) & reachable_mask(graph, labels)
                eligs.append(elig.astype(np.uint8))
                digests.append(csr_digest(graph))
                if component_init and len(rb.insert_ids) and not rb.is_empty:
                    lab = find_components(IntraBatchGraph.build(rb.insert_ids, rb.insert_edges(), tv))
                    intra.append(np.stack([lab.vertices, lab.parent, lab.component_id]))
                else:
                    intra.append(np.zeros((3, 0), dtype=np.int64))
        if c == 0:
            csr = graph.csr()
            final = (csr.indptr, csr.indices, csr.weights, csr.degrees)
    arrs = pack_batches(batches)
    arrs.update(
        cfg=np.array([delta, math.nan if tau == "auto" else float(tau),
                      0 if max_iterations is None else max_iterations,
                      int(component_init), 0 if mode == "parallel_jacobi" else 1, num_classes],
                     dtype=np.float64),
        slots=np.array(slots, dtype=np.int64),
        f=np.concatenate([np.concatenate(fc) for fc in f_cols]),
        rep_i=rep_i, rep_mc=rep_mc, tau=np.array(taus),
        elig=np.concatenate(eligs), csr_sha=np.array(digests),
        intra=np.concatenate(intra, axis=1) if intra else np.zeros((3, 0), np.int64),
        intra_off=np.cumsum([0] + [x.shape[1] for x in intra]),
        final_indptr=final[0], final_indices=final[1], final_weights=final[2],
        final_degrees=final[3],
    )
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **arrs)
    print(f"{name}: {nb} batches, |V|={slots[-1]}, cols={ncol}, "
          f"iters={rep_i[:, :, 0].sum()}, {os.path.getsize(path)} bytes")


def pack_batches(batches):
    cat = lambda key, dt: np.concatenate([np.asarray(getattr(b, key), dt) for b in batches])  # noqa
    off = lambda key: np.cumsum([0] + [len(getattr(b, key)) for b in batches])  # noqa
    return dict(
        b_t=np.array([b.t for b in batches], dtype=np.int64),
        b_ins=cat("insert_ids", np.int64), b_gt=cat("insert_gt", np.int8),
        b_owner=cat("edge_owner", np.int64), b_other=cat("edge_other", np.int64),
        b_w=cat("edge_w", np.float64), b_del=cat("deletes", np.int64),
        b_ins_off=off("insert_ids"), b_edge_off=off("edge_owner"), b_del_off=off("deletes"),
    )


def ref_stream(n, deg, seed, batch, fr=(0.90, 0.01, 0.09), init_gt=4, labeled=0.05):
    from dynlp.builder import SyntheticSpec, erdos_renyi
    from dynlp.stream import StreamSpec, make_stream

    data = erdos_renyi(SyntheticSpec(n=n, avg_degree=deg, seed=seed, labeled_fraction=labeled))
    s = make_stream(data.n, data.edges, data.gt_ids, data.gt_classes,
                    StreamSpec(batch_size=batch, seed=seed, insert_fraction=fr[0],
                               gt_fraction=fr[1], delete_fraction=fr[2], initial_gt_count=init_gt))
    return s.batches


def adversarial_batches():
    R = OwnBatch.from_records
    return [
        R([(0, [], 0), (1, [], 1), (2, [(2, 0, 1.0), (2, 1, 2.0)], None),
           (3, [(3, 2, 0.5), (3, 2, 0.25), (3, 0, 0.0)], None),   # parallel edge + zero weight
           (4, [], None),                                          # isolated, unreachable
           (5, [(5, 4, 1.0)], None)], t=0),                        # unreachable pair
        R([(6, [(6, 3, 1.0), (6, 5, 0.7), (6, 7, 0.9)], None),
           (7, [(7, 6, 0.1), (7, 1, 3.0)], None),                  # reverse dup across records
           (8, [(8, 7, 2.0), (8, 2, 1e-3)], 0)], t=1),
        R(t=2),                                                    # empty batch
        R([(9, [(9, 8, 1.0), (9, 4, 2.0)], None)], deletes=[1], t=3),  # delete a GT vertex
        R([(10, [(10, 9, 0.6), (10, 6, 0.6)], 1), (11, [(11, 10, 0.6)], None)],
          deletes=[2, 5], t=4),
        R(deletes=[0, 8], t=5),                                    # cut all class-0 seeds
        R([(12, [(12, 3, 4.0), (12, 11, 1.0)], 0), (13, [(13, 12, 1.0)], None)], t=6),
    ]


def blob_stream(n, dim, k, C, seed, batch, fr):
    bl = streams.make_blobs(n, dim, C, seed)
    edges = streams.knn_graph_exact(bl.x, k)
    gt = streams.stratified_seeds(bl.classes, 0.02, seed)
    return streams.phased_stream(n, edges, bl.classes, gt, batch, seed, insert_fraction=fr[0],
                                 gt_fraction=fr[1], delete_fraction=fr[2], initial_gt=2 * C).batches


def kernel_cases():
    from dynlp.kernels import _csr

    rng = np.random.default_rng(1234)
    out = {}
    for seed in range(4):
        n = 120
        m = 360
        a = rng.integers(0, n, m)
        b = rng.integers(0, n, m)
        ok = a != b
        edges = EdgeList(a[ok], b[ok], rng.uniform(0.05, 1.0, ok.sum()))
        if seed == 3:  # zero-weight rows: kernel-detected isolated vertices
            edges.w[:20] = 0.0
        g = DynamicGraph.from_edge_list(n, edges, merge=(seed != 2))
        csr = g.csr()
        gt = np.full(n, -1, np.int8)
        gt[rng.choice(n, 10, replace=False)] = rng.integers(0, 2, 10)
        f = np.where(gt >= 0, gt.astype(np.float64), rng.uniform(0, 1, n))
        frontier = np.flatnonzero(gt < 0).astype(np.int64)
        if seed == 1:
            frontier = np.concatenate([frontier, frontier[:7]])  # duplicates
        vals = np.empty(len(frontier))
        deltas = np.empty(len(frontier))
        _csr.jacobi_step(csr.indptr, csr.indices, csr.weights, gt, f, frontier, vals, deltas, 1)
        elig = ((gt < 0) & (np.diff(csr.indptr) > 0)).astype(np.uint8)
        if seed == 3:
            elig[:] = (gt < 0)  # let zero-weight rows in so the sentinel path runs
        f2 = f.copy()
        e2 = elig.copy()
        it, upd, mc, warn, left = _csr.jacobi_run(csr.indptr, csr.indices, csr.weights, gt, f2,
                                                  frontier, e2, 1e-7, 10_000 if seed != 0 else 5, 1)
        f3 = f.copy()
        d3 = np.empty(len(frontier))
        _csr.gauss_seidel_step(csr.indptr, csr.indices, csr.weights, gt, f3, frontier, d3)
        p = f"k{seed}_"
        out.update({p + "indptr": csr.indptr, p + "indices": csr.indices,
                    p + "weights": csr.weights, p + "gt": gt, p + "f": f,
                    p + "frontier": frontier, p + "vals": vals, p + "deltas": deltas,
                    p + "elig": elig, p + "run_f": f2, p + "run_elig": e2,
                    p + "run_out": np.array([it, upd, warn, len(left)], dtype=np.int64),
                    p + "run_mc": np.array([mc]), p + "run_left": np.sort(left),
                    p + "gs_f": f3, p + "gs_deltas": d3})
    path = os.path.join(HERE, "kernels.npz")
    np.savez_compressed(path, **out)
    print("kernels:", os.path.getsize(path), "bytes")


def pairwise_cases():
    rng = np.random.default_rng(99)
    sizes = [0, 1, 3, 7, 8, 9, 16, 17, 127, 128, 129, 130, 255, 1000, 4097, 100_003, 1_000_001]
    vals = []
    arrs = []
    for n in sizes:
        a = rng.uniform(0, 1, n) * rng.choice([1e-3, 1.0, 1e3], n)
        vals.append(float(a.mean()) if n else 0.0)
        arrs.append(a)
    np.savez_compressed(os.path.join(HERE, "pairwise.npz"), sizes=np.array(sizes),
                        means=np.array(vals), seed=np.array([99]))
    print("pairwise: sizes", sizes)


if __name__ == "__main__":
    run_case("er_mixed", ref_stream(300, 5, 9, 40), delta=1e-6)
    run_case("er_heavy_delete", ref_stream(400, 6, 3, 50, fr=(0.6, 0.02, 0.38)), delta=1e-5,
             tau=0.5)
    run_case("blobs3_mixed", blob_stream(500, 8, 6, 3, 0, 60, (0.70, 0.02, 0.28)), num_classes=3,
             delta=1e-6)
    run_case("blobs2_insert", blob_stream(600, 16, 10, 2, 1, 100, (0.98, 0.02, 0.0)), delta=1e-4)
    adv = adversarial_batches()
    run_case("adversarial", adv, delta=1e-9)
    run_case("adversarial_noinit_budget", adv, delta=1e-9, component_init=False, max_iterations=3)
    run_case("er_gauss_seidel", ref_stream(200, 5, 4, 30), delta=1e-6, mode="sequential_gauss_seidel")
    kernel_cases()
    pairwise_cases()
