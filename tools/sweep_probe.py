"""Time one full ItLP sweep (every active row, all label columns) of the C2
graph at |V| ~ 0.99M: the LP kernel's throughput without frontier dynamics.
Diagnostic tool; DLP_LIB_PATH selects a library variant."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2604_06596_b200.batch import BatchUpdate  # noqa: E402
from paper_2604_06596_b200.engine import DynamicGraph, EngineConfig, LabelState, apply_batch, itlp_batch_solve  # noqa: E402

cfg = dict(bench.CONFIGS["c2"])
batches, _ = bench.make_stream(cfg, "cuda:0")
g, lab = DynamicGraph(0, num_classes=10), LabelState()
g.reserve(sum(len(b.insert_ids) for b in batches), sum(len(b.edge_owner) for b in batches))
ecfg = EngineConfig(delta=1e-4)
for b in batches[:99]:
    apply_batch(g, lab, b, ecfg)
empty = BatchUpdate(t=999, insert_ids=np.empty(0, np.int64), insert_gt=np.empty(0, np.int8),
                    edge_owner=np.empty(0, np.int64), edge_other=np.empty(0, np.int64), edge_w=np.empty(0),
                    deletes=np.empty(0, np.int64))
one = EngineConfig(delta=1e9)  # converged after one sweep
res = []
for r in range(5):
    _, reps = itlp_batch_solve(g, lab, empty, one)
    rep = reps[0]
    res.append((rep.lp_kernel_ms, rep.lp_union_rows, rep.lp_union_entries, rep.iterations))
best = min(res)
tr = os.environ.get("DLP_LP_TRACE")
if tr and os.path.exists(tr):
    print([ln.strip() for ln in open(tr) if ln.startswith("#")][-1])
print(f"sweep: {best[0]:.3f} ms, rows {best[1]}, entries {best[2]}, "
      f"{best[2] / best[0] / 1e6:.2f} G entries/s  all={[round(x[0], 3) for x in res]}")
