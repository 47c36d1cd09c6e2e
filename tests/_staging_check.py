"""Subprocess body of test_ingestion_pipeline_staging_growth: with the staging
floor at 0 (DLP_STAGE_FLOOR_MB=0, set by the caller) every batch of a stream
whose batches grow 8x outgrows the pinned / device staging slots, so the
pipelined path reallocates both slots between batches; reports and labels must
equal the unpipelined run bit for bit."""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

from paper_2604_06596_b200 import streams  # noqa: E402
from paper_2604_06596_b200.engine import DynamicGraph, EngineConfig, LabelState, run_batches  # noqa: E402


def main():
    bl = streams.make_blobs(6000, 16, 3, 4)
    e = streams.knn_graph_exact(bl.x, 8)
    gt = streams.stratified_seeds(bl.classes, 0.02, 4)
    phases = [(2, 50, 0.98, 0.02, 0.0), (2, 400, 0.98, 0.02, 0.0), (None, 1600, 0.8, 0.02, 0.18)]
    s = streams.phased_stream(6000, e, bl.classes, gt, 50, 4, phases=phases, initial_gt=6)
    cfg = EngineConfig(delta=1e-5)
    g1, l1 = DynamicGraph(0, num_classes=3), LabelState()
    r1 = run_batches(g1, l1, s.batches, cfg, pipelined=False)
    g2, l2 = DynamicGraph(0, num_classes=3), LabelState()
    r2 = run_batches(g2, l2, s.batches, cfg, pipelined=True)
    for t, (a, b) in enumerate(zip(r1, r2)):
        ka = [(x.iterations, x.updates, x.max_change) for x in a]
        kb = [(x.iterations, x.updates, x.max_change) for x in b]
        assert ka == kb, f"batch {t}: {ka} != {kb}"
    assert l1.F.tobytes() == l2.F.tobytes()
    g1.close()
    g2.close()
    print("ok", len(s.batches))


if __name__ == "__main__":
    main()
