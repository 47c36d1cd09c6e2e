"""Generate tests/golden/knn_*.npz by running the REAL reference knn_graph
(builder.py:42-92) in this container (oracle.load_reference()).

Cases: the reference's own known-answer tests (tests/test_builder.py:30-47:
identical vectors -> {(0,1),(0,2)}, orthogonal prune -> empty, affine 0.5),
its brute-force oracle case shape (40 x 6, k=3, affine), blob data of the
C1 shape (features 16-dim, k=10) and a duplicate-row tie case.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import load_reference  # noqa: E402
from paper_2604_06596_b200 import streams  # noqa: E402

assert load_reference() is not None, "reference not importable"
from dynlp.builder import FeatureMatrix, knn_graph  # noqa: E402


def cases():
    rng = np.random.default_rng(0)
    yield "triangle", np.array([[1.0, 2.0]] * 3), 1, "prune"
    yield "eye_prune", np.eye(3), 1, "prune"
    yield "eye_affine", np.eye(3), 1, "affine"
    for s in range(3):
        yield f"normal40_s{s}", np.random.default_rng(s).normal(size=(40, 6)), 3, "affine"
    yield "normal300_k7", rng.normal(size=(300, 12)), 7, "prune"
    dup = rng.normal(size=(200, 8))
    dup[100:150] = dup[:50]  # exact duplicate rows: equal sims, ties to the lower id
    yield "dups200", dup, 5, "affine"
    # blob features are regenerated from (n, dim, classes, seed) by the tests
    yield "blobs2000_k10", ("blobs", 2000, 16, 3, 0), 10, "prune"
    yield "blobs3000_d96_k16", ("blobs", 3000, 96, 10, 1), 16, "affine"


if __name__ == "__main__":
    out = {}
    for name, x, k, mode in cases():
        spec = None
        if isinstance(x, tuple):
            spec = np.array(x[1:], dtype=np.int64)
            x = streams.make_blobs(*x[1:]).x
        e = knn_graph(FeatureMatrix(x), k, similarity_mode=mode)
        out[name] = dict(k=k, mode=mode, u=np.asarray(e.u), v=np.asarray(e.v), w=np.asarray(e.w))
        if spec is None:
            out[name]["x"] = x
        else:
            out[name]["blobs"] = spec
        print(name, x.shape, k, mode, len(e.u))
    np.savez_compressed(os.path.join(HERE, "knn_reference.npz"),
                        **{f"{n}__{f}": (np.asarray(v) if f != "mode" else np.array(v))
                           for n, d in out.items() for f, v in d.items()})
