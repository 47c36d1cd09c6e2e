"""Subprocess body of test_row_class_paths: run a ten-column blob stream with
low row-class thresholds (DLP_LONG_ROW / DLP_HUB_ROW set by the caller) so the
short, long and hub (CTA-cooperative) paths of the LP kernel all run in the
same rounds, and compare every report and label bit with the C oracle."""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

from oracle import OracleEngine  # noqa: E402
from paper_2604_06596_b200 import streams  # noqa: E402
from paper_2604_06596_b200.engine import DynamicGraph, EngineConfig, LabelState, apply_batch  # noqa: E402


def main():
    ncls = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    bl = streams.make_blobs(3000, 32, max(ncls, 2), 5)
    e = streams.knn_graph_exact(bl.x, 12)
    gt = streams.stratified_seeds(bl.classes, 0.01, 5)
    s = streams.phased_stream(3000, e, bl.classes, gt, 400, 5, 0.8, 0.01, 0.19, initial_gt=2 * ncls)
    g, lab = DynamicGraph(0, num_classes=ncls), LabelState()
    orc = OracleEngine(ncls, threads=4)
    for t, b in enumerate(s.batches):
        lab, rep = apply_batch(g, lab, b, EngineConfig(delta=1e-5))
        reps = rep if isinstance(rep, list) else [rep]
        for c, (r, o) in enumerate(zip(reps, orc.apply_batch(b, delta=1e-5))):
            got = (r.iterations, r.updates, r.max_change, r.edges_traversed)
            want = (o.iterations, o.updates, o.max_change, o.edges_traversed)
            assert got == want, f"batch {t} column {c}: {got} != {want}"
        f, _ = orc.labels()
        assert lab.F.tobytes() == f.tobytes(), f"batch {t}: labels differ"
    g.close()
    print("ok", len(s.batches))


if __name__ == "__main__":
    main()
