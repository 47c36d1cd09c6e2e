import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
from oracle import OracleEngine
from paper_2604_06596_b200 import streams
from paper_2604_06596_b200.engine import DynamicGraph, LabelState, EngineConfig, apply_batch
bl = streams.make_blobs(4000, 32, 10, 7)
e = streams.knn_graph_exact(bl.x, 10)
gt = streams.stratified_seeds(bl.classes, 0.01, 7)
s = streams.phased_stream(4000, e, bl.classes, gt, 500, 7, 0.99, 0.01, 0.0, initial_gt=20)
deg = np.bincount(e.u, minlength=4000) + np.bincount(e.v, minlength=4000)
print("max degree", deg.max())
orc = OracleEngine(10, threads=4)
ores = [orc.apply_batch(b, delta=1e-4) for b in s.batches]
for trial in range(2):
    g, lab = DynamicGraph(0, num_classes=10), LabelState()
    for t, b in enumerate(s.batches):
        lab, rep = apply_batch(g, lab, b, EngineConfig(delta=1e-4))
        bad = [(c, r.iterations, r.updates, o.iterations, o.updates) for c, (r, o) in enumerate(zip(rep, ores[t]))
               if (r.iterations, r.updates) != (o.iterations, o.updates)]
        if bad:
            print("trial", trial, "batch", t, "mismatch cols", bad)
            break
    else:
        print("trial", trial, "ok")
    g.close()
