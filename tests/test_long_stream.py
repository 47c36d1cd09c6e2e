"""North-star parity run: >= 100 mixed insert/delete batches at >= 50k alive
vertices with 10 one-vs-rest label columns, the CUDA engine against the C
oracle (itself pinned bitwise to the compiled reference by test_oracle.py)
batch by batch: every IterationReport field, tau, the eligible mask and the
bytes of every label column.

Stream rules follow the reference's make_stream (stream.py:56-183): a
bootstrap phase of insert batches, then mixed batches of 69% unlabeled + 1%
ground-truth inserts and 30% deletes (SURVEY.md §8(d) D-2 C3 recipe, scaled).
The blobs overlap (centre spread 2 sigma) so components merge and split and
the ten columns evolve differently."""

import numpy as np
import pytest

from golden_io import report_tuple
from oracle import OracleEngine
from paper_2604_06596_b200 import streams


def _stream(n_boot=50, n_mixed=100, bs=1000, classes=10, seed=7, device="cpu"):
    n = n_boot * bs + n_mixed * bs  # enough points for both phases
    bl = streams.make_blobs(n, 16, classes, seed, spread=2.0)
    edges = streams.knn_graph_torch64(bl.x, 10, device=device)
    gt = streams.stratified_seeds(bl.classes, 0.01, seed)
    s = streams.phased_stream(n, edges, bl.classes, gt, bs, seed, 0.69, 0.01, 0.30, initial_gt=2 * classes,
                              phases=[(n_boot, bs, 0.99, 0.01, 0.0), (n_mixed, bs, 0.69, 0.01, 0.30)])
    return s.batches


def test_phased_stream_shape():
    b = _stream(n_boot=3, n_mixed=4, bs=200, classes=4)
    assert len(b) == 1 + 3 + 4
    assert all(len(x.deletes) == 0 for x in b[:4])
    assert all(len(x.deletes) == 60 and len(x.insert_ids) == 140 for x in b[4:])


@pytest.mark.gpu
@pytest.mark.slow
def test_100_mixed_batches_ten_columns_bitwise(gpu_device):
    import os

    from paper_2604_06596_b200.engine import DynamicGraph, EngineConfig, LabelState, apply_batch

    batches = _stream(device="cuda")
    mixed = [b for b in batches if len(b.deletes)]
    assert len(mixed) >= 100
    g, lab = DynamicGraph(0, num_classes=10), LabelState()
    orc = OracleEngine(10, threads=os.cpu_count() or 4)
    cfg = EngineConfig(delta=1e-4)
    min_alive = None
    for t, b in enumerate(batches):
        lab, rep = apply_batch(g, lab, b, cfg)
        orep = orc.apply_batch(b, delta=1e-4)
        for c, (r, o) in enumerate(zip(rep, orep)):
            assert report_tuple(r) == report_tuple(o), f"batch {t} column {c}: {r} vs {o}"
            assert r.max_change == o.max_change, f"batch {t} column {c}"
            assert r.edges_traversed == o.edges_traversed, f"batch {t} column {c}"
        assert g.last_tau == orc.last_tau, f"batch {t}: tau"
        assert np.array_equal(g.eligible(), orc.eligible()), f"batch {t}: eligible"
        F = lab.F
        of, _ = orc.labels()
        assert F.tobytes() == of.tobytes(), f"batch {t}: labels differ (max abs {np.abs(F - of).max():.3g})"
        if len(b.deletes):
            min_alive = g.num_alive if min_alive is None else min(min_alive, g.num_alive)
    assert min_alive >= 50_000
    g.close()
