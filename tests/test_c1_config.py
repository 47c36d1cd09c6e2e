"""BASELINE.json config 1 end to end against the real reference
(tests/golden/c1_reference.npz, made by make_c1_golden.py): the C1 stream
(blobs 10k x 16, 3 classes, kNN k=10, 1% seeds, batches of 500) built with
the B200 k-NN builder equals the reference-built stream edge for edge, and
the B200 engine's 3 one-vs-rest columns reproduce every report and every
label bit of the reference's per-column runs."""

import hashlib
import os

import numpy as np
import pytest

from paper_2604_06596_b200.batch import BatchUpdate

PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "c1_reference.npz")
Z = np.load(PATH)


def _batches():
    io, eo, do = Z["b_ins_off"], Z["b_edge_off"], Z["b_del_off"]
    return [BatchUpdate(t=int(Z["b_t"][t]), insert_ids=Z["b_ins"][io[t]:io[t + 1]],
                        insert_gt=Z["b_gt"][io[t]:io[t + 1]], edge_owner=Z["b_owner"][eo[t]:eo[t + 1]],
                        edge_other=Z["b_other"][eo[t]:eo[t + 1]], edge_w=Z["b_w"][eo[t]:eo[t + 1]],
                        deletes=Z["b_del"][do[t]:do[t + 1]]) for t in range(len(Z["b_t"]))]


def test_c1_golden_shape():
    b = _batches()
    assert len(b) == Z["reps"].shape[0] and Z["reps"].shape[1] == 3
    assert sum(len(x.insert_ids) for x in b) == 10_000


@pytest.mark.gpu
def test_c1_stream_from_b200_knn_matches_reference(gpu_device):
    from paper_2604_06596_b200 import streams
    from paper_2604_06596_b200.knn import knn_graph

    bl = streams.make_blobs(10_000, 16, 3, 0)
    e = knn_graph(bl.x, 10)
    gt = streams.stratified_seeds(bl.classes, 0.01, 0)
    s = streams.phased_stream(10_000, e, bl.classes, gt, 500, 0, 0.99, 0.01, 0.0, initial_gt=6)
    ref = _batches()
    assert len(s.batches) == len(ref)
    for a, b in zip(s.batches, ref):
        assert np.array_equal(a.insert_ids, b.insert_ids) and np.array_equal(a.insert_gt, b.insert_gt)
        assert np.array_equal(a.edge_owner, b.edge_owner) and np.array_equal(a.edge_other, b.edge_other)
        assert np.allclose(a.edge_w, b.edge_w, rtol=0, atol=1e-12)


@pytest.mark.gpu
def test_c1_engine_matches_reference(gpu_device):
    from paper_2604_06596_b200.engine import DynamicGraph, EngineConfig, LabelState, apply_batch

    g, lab = DynamicGraph(0, num_classes=3), LabelState()
    cfg = EngineConfig(delta=1e-4)
    for t, b in enumerate(_batches()):
        lab, reps = apply_batch(g, lab, b, cfg)
        F = lab.F
        for c, r in enumerate(reps):
            want = Z["reps"][t, c]
            got = (r.iterations, r.updates, int(r.converged), r.warnings, r.isolated_pinned, r.unreachable_pinned)
            assert got == tuple(int(x) for x in want[:6]), f"batch {t} column {c}: {got} vs {want}"
            assert r.max_change == want[6]
            assert hashlib.sha256(F[c].tobytes()).hexdigest() == Z["sha"][t, c], f"batch {t} column {c}"
    assert lab.F.tobytes() == Z["final_f"].tobytes()
    g.close()
