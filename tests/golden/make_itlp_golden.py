"""Generate tests/golden/itlp_reference.npz by running the REAL reference
``baselines.itlp_batch_solve`` (baselines.py:236-253) in this container.

Streams: an ER stream with deletes (reference make_stream), the adversarial
stream of make_golden.py (isolated / unreachable vertices, deleted seeds,
empty batch) and a 3-class blob stream (one-vs-rest reference runs, ground
truth remapped per column as in make_golden.py).  Per batch: f of every
column and the IterationReport fields.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import make_golden as mg  # noqa: E402  (imports the reference)
from dynlp.baselines import itlp_batch_solve  # noqa: E402
from dynlp.engine import EngineConfig  # noqa: E402
from dynlp.graph import DynamicGraph  # noqa: E402
from dynlp.labels import LabelState  # noqa: E402


def run(name, batches, num_classes=2, delta=1e-6, max_iterations=None):
    ncol = 1 if num_classes <= 2 else num_classes
    fs, reps = [], []
    graphs = [(DynamicGraph(), LabelState()) for _ in range(ncol)]
    cfg = EngineConfig(delta=delta, max_iterations=max_iterations, threads=1)
    for b in batches:
        fcol, rcol = [], []
        for c, (g, lab) in enumerate(graphs):
            rb = mg.to_ref(b if ncol == 1 else mg.remap(b, c))
            lab, rep = itlp_batch_solve(g, lab, rb, cfg)
            graphs[c] = (g, lab)
            fcol.append(lab.f[: g.num_slots].copy())
            rcol.append([rep.iterations, rep.updates, int(rep.converged), rep.warnings, rep.isolated_pinned,
                         rep.unreachable_pinned, rep.max_change])
        fs.append(np.stack(fcol))
        reps.append(rcol)
    out = dict(mg.pack_batches(batches))
    out["f_off"] = np.cumsum([0] + [f.size for f in fs])
    out["f"] = np.concatenate([f.ravel() for f in fs])
    out["reps"] = np.array(reps, dtype=np.float64)
    out["meta"] = np.array([num_classes, delta, -1 if max_iterations is None else max_iterations])
    return {f"{name}__{k}": v for k, v in out.items()}


if __name__ == "__main__":
    d = {}
    d.update(run("er_mixed", mg.ref_stream(600, 6, 3, 80)))
    d.update(run("adversarial", mg.adversarial_batches()))
    d.update(run("adversarial_budget", mg.adversarial_batches(), max_iterations=3))
    d.update(run("blobs3", mg.blob_stream(400, 8, 6, 3, 1, 60, (0.80, 0.02, 0.18)), num_classes=3, delta=1e-5))
    np.savez_compressed(os.path.join(HERE, "itlp_reference.npz"), **d)
    print(sorted({k.split("__")[0] for k in d}))
