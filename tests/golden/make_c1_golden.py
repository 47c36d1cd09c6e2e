"""Golden record of BASELINE.json config 1 (C1) through the REAL reference:
Gaussian blobs 10k x 16, 3 classes, cosine kNN k=10 (the reference's own
knn_graph), 1% stratified seeds, insert batches of 500 (make_stream rules),
delta = 1e-4.  The reference is binary (labels.py:42-43), so each class
column is an independent reference run with ground truth remapped (one vs
rest).  Records per batch and column the IterationReport fields and a
SHA-256 of the label bytes, plus the final label matrix."""
import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import make_golden as mg  # noqa: E402  (imports the reference)
from dynlp.builder import FeatureMatrix, knn_graph  # noqa: E402
from dynlp.engine import EngineConfig, apply_batch  # noqa: E402
from dynlp.graph import DynamicGraph  # noqa: E402
from dynlp.labels import LabelState  # noqa: E402

from paper_2604_06596_b200 import streams  # noqa: E402
from paper_2604_06596_b200.batch import EdgeList  # noqa: E402


def c1_stream():
    bl = streams.make_blobs(10_000, 16, 3, 0)
    e = knn_graph(FeatureMatrix(bl.x), 10)
    edges = EdgeList(np.asarray(e.u), np.asarray(e.v), np.asarray(e.w))
    gt = streams.stratified_seeds(bl.classes, 0.01, 0)
    s = streams.phased_stream(10_000, edges, bl.classes, gt, 500, 0, 0.99, 0.01, 0.0, initial_gt=6)
    return s.batches, s.classes


if __name__ == "__main__":
    batches, classes = c1_stream()
    cfg = EngineConfig(delta=1e-4, threads=1)
    nb, C = len(batches), 3
    reps = np.zeros((nb, C, 7), dtype=np.float64)
    sha = np.empty((nb, C), dtype="<U64")
    finals = []
    for c in range(C):
        g, lab = DynamicGraph(), LabelState()
        for t, b in enumerate(batches):
            lab, r = apply_batch(g, lab, mg.to_ref(mg.remap(b, c)), cfg)
            reps[t, c] = [r.iterations, r.updates, int(r.converged), r.warnings, r.isolated_pinned,
                          r.unreachable_pinned, r.max_change]
            sha[t, c] = hashlib.sha256(lab.f[: g.num_slots].tobytes()).hexdigest()
        finals.append(lab.f[: g.num_slots].copy())
    out = dict(mg.pack_batches(batches))
    out.update(reps=reps, sha=sha, final_f=np.stack(finals), classes=classes)
    np.savez_compressed(os.path.join(HERE, "c1_reference.npz"), **out)
    print(nb, "batches", reps[:, :, 0].sum(), "iterations", os.path.getsize(os.path.join(HERE, "c1_reference.npz")))
