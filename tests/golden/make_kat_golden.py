"""Known-answer fixtures from the reference's own engine tests (this container only).

    python tests/golden/make_kat_golden.py   ->  tests/golden/kats.npz

Each scenario restates one of the reference's engine-level known-answer tests
(/root/reference/pkg/tests/test_engine.py) as a batch stream, runs the REAL
reference (compiled backend, oracle.load_reference()) over it and records:

* the stream (flattened BatchUpdate arrays), the EngineConfig of every batch,
* per batch: the IterationReport fields and f (all slots),
* the closed-form harmonic labels of the final state (baselines.harmonic_solve,
  baselines.py:163-190) -- the accuracy oracle of test_engine.py:154-162, 190-192.

Random instances come from the reference's own generator
(tests/helpers.py:67-95, random_connected_instance) so the graphs are the
reference's test graphs exactly.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import load_reference  # noqa: E402

assert load_reference() is not None, "reference not importable"
sys.path.insert(0, "/root/reference/pkg/tests")
import dynlp.kernels as rk  # noqa: E402

assert rk.BACKEND == "compiled", rk.BACKEND
from dynlp.baselines import harmonic_solve, stlp_solve  # noqa: E402
from dynlp.errors import ValidationError  # noqa: E402
from dynlp.engine import EngineConfig, apply_batch  # noqa: E402
from dynlp.graph import BatchUpdate, DynamicGraph  # noqa: E402
from dynlp.labels import LabelState  # noqa: E402
from helpers import graph_as_batch, random_connected_instance  # noqa: E402  (reference tests/helpers.py)


def rec(inserts=(), deletes=(), t=0):
    return BatchUpdate.from_records(list(inserts), deletes=list(deletes), t=t)


def scenarios():
    """name -> (list of (BatchUpdate, EngineConfig kwargs), reference test cited)."""
    out = {}
    conv = dict(delta=1e-9, max_iterations=500_000)
    # test_engine.py:131-140 empty batch is a no-op
    out["empty_batch"] = [
        (graph_as_batch(4, [(0, 1, 1.0), (1, 2, 1.0), (2, 3, 1.0)], {0: 0, 3: 1}), conv),
        (rec(t=9), {}),
    ]
    # test_engine.py:165-198 structural trace: deletes, inserts, two new components
    pre = rec([(0, [], 0), (1, [], 0), (2, [], 1), (3, [], 1), (4, [(4, 0, 1.0), (4, 5, 1.0)], None),
               (5, [(5, 2, 1.0)], None), (6, [(6, 5, 1.0)], None)])
    bat = rec([(7, [(7, 8, 0.9), (7, 0, 2.0)], None), (8, [(8, 1, 1.0)], None),
               (9, [(9, 3, 3.0), (9, 5, 1.0)], None)], deletes=[6], t=1)
    out["structural_trace"] = [(pre, dict(delta=1e-9)), (bat, dict(delta=1e-9, tau=0.5))]
    # test_engine.py:200-208 a new ground-truth seed pulls its neighbour
    out["new_gt_seed"] = [
        (graph_as_batch(3, [(0, 1, 1.0), (1, 2, 1.0)], {0: 0, 2: 1}), conv),
        (rec([(3, [(3, 1, 10.0)], 1)], t=1), dict(delta=1e-9)),
    ]
    # test_engine.py:210-218 deleting a ground-truth vertex
    out["delete_gt"] = [
        (graph_as_batch(4, [(0, 1, 1.0), (1, 2, 1.0), (1, 3, 1.0)], {0: 0, 2: 1, 3: 1}), conv),
        (rec(deletes=[2], t=1), dict(delta=1e-9)),
    ]
    # test_engine.py:220-238 a vertex cut off from every seed is pinned to 0.5
    out["unreachable_pin"] = [
        (graph_as_batch(5, [(0, 1, 1.0), (1, 2, 1.0), (2, 3, 1.0), (3, 4, 1.0)], {0: 0, 4: 1}), conv),
        (rec(deletes=[0], t=1), {}),
        (rec(deletes=[2], t=2), {}),
    ]
    # test_engine.py:240-248 iteration budget -> not converged, iterations == budget
    pairs, gt = random_connected_instance(np.random.default_rng(11), 60, 5)
    out["budget_two"] = [(graph_as_batch(60, pairs, gt), dict(delta=1e-12, max_iterations=2))]
    # test_engine.py:154-162 a single batch converges to the harmonic solution
    pairs, gt = random_connected_instance(np.random.default_rng(3), 80, 5)
    out["single_batch_harmonic"] = [(graph_as_batch(80, pairs, gt), conv)]
    # test_engine.py:252-262 fixed-point residuals at convergence (delta 1e-5)
    for seed in range(5):
        pairs, gt = random_connected_instance(np.random.default_rng(seed), 70, 4)
        out[f"fixed_point_{seed}"] = [(graph_as_batch(70, pairs, gt), dict(delta=1e-5, max_iterations=500_000))]
    return out


REPORT_FIELDS = ("iterations", "updates", "max_change", "converged", "warnings", "isolated_pinned",
                 "unreachable_pinned")


def kernel_cases(data):
    """test_kernels.py:14-20 random_state(seed) for seeds 0..4 (n=80, degree 5)
    and the compiled backend's jacobi_step / jacobi_run / gauss_seidel_step
    outputs on it (test_kernels.py:23-77)."""
    from helpers import build_graph

    for seed in range(5):
        rng = np.random.default_rng(seed)
        pairs, gt = random_connected_instance(rng, 80, 5)
        graph, labels = build_graph(80, pairs, gt)
        unl = labels.unlabeled_ids(graph)
        labels.f[unl] = rng.uniform(0, 1, len(unl))
        csr = graph.csr()
        p = f"kern{seed}/"
        data[p + "indptr"], data[p + "indices"], data[p + "weights"] = csr.indptr, csr.indices, csr.weights
        data[p + "gt"], data[p + "f"], data[p + "unl"] = labels.gt.copy(), labels.f.copy(), unl
        vals, deltas = np.empty(len(unl)), np.empty(len(unl))
        rk.jacobi_step(csr.indptr, csr.indices, csr.weights, labels.gt, labels.f, unl, vals, deltas, 1)
        data[p + "step_vals"], data[p + "step_deltas"] = vals, deltas
        f = labels.f.copy()
        elig = (graph.alive & (labels.gt[: graph.num_slots] == -1) & (csr.degrees > 0)).view(np.uint8).copy()
        data[p + "eligible"] = elig.copy()
        it, upd, mc, warn, left = rk.jacobi_run(csr.indptr, csr.indices, csr.weights, labels.gt, f, unl, elig,
                                                1e-6, 10_000, 1)
        data[p + "run_out"] = np.asarray([it, upd, mc, warn, len(left)], np.float64)
        data[p + "run_f"], data[p + "run_elig"] = f, elig
        f = labels.f.copy()
        d = np.empty(len(unl))
        rk.gauss_seidel_step(csr.indptr, csr.indices, csr.weights, labels.gt, f, unl, d)
        data[p + "gs_f"], data[p + "gs_deltas"] = f, d


def main():
    data = {}
    names = []
    for name, steps in scenarios().items():
        names.append(name)
        g, lab = DynamicGraph(), LabelState()
        cols = {k: [] for k in ("ids", "gt", "own", "oth", "w", "dels")}
        offs = {k: [0] for k in ("io", "eo", "do")}
        cfgs, reps, fs = [], [], []
        for b, kw in steps:
            cfg = EngineConfig(**kw)
            lab, r = apply_batch(g, lab, b, cfg)
            cols["ids"].append(b.insert_ids)
            cols["gt"].append(b.insert_gt)
            cols["own"].append(b.edge_owner)
            cols["oth"].append(b.edge_other)
            cols["w"].append(b.edge_w)
            cols["dels"].append(b.deletes)
            offs["io"].append(offs["io"][-1] + len(b.insert_ids))
            offs["eo"].append(offs["eo"][-1] + len(b.edge_owner))
            offs["do"].append(offs["do"][-1] + len(b.deletes))
            tau = kw.get("tau", "auto")
            cfgs.append([cfg.delta, np.nan if tau == "auto" else float(tau),
                         -1 if cfg.max_iterations is None else cfg.max_iterations, int(b.t)])
            reps.append([float(getattr(r, f)) for f in REPORT_FIELDS])
            f = np.full(g.num_slots, 0.5)
            f[:] = lab.f[: g.num_slots]
            fs.append(f)
        p = name + "/"
        for k, v in cols.items():
            data[p + k] = np.concatenate(v) if v else np.zeros(0)
        for k, v in offs.items():
            data[p + k] = np.asarray(v, np.int64)
        data[p + "cfg"] = np.asarray(cfgs, np.float64)
        data[p + "reports"] = np.asarray(reps, np.float64)
        data[p + "f_n"] = np.asarray([len(x) for x in fs], np.int64)
        data[p + "f"] = np.concatenate(fs)
        data[p + "alive"] = g.alive.astype(np.uint8)
        data[p + "gt_final"] = lab.gt[: g.num_slots].copy()
        data[p + "harmonic"] = harmonic_solve(g, lab)
        try:  # baselines.py:290-318 (short-circuit contraction; needs both classes)
            data[p + "stlp"] = stlp_solve(g, lab.copy()).f[: g.num_slots].copy()
        except ValidationError:
            data[p + "stlp"] = np.full(g.num_slots, np.nan)
    kernel_cases(data)
    data["names"] = np.asarray(names)
    data["report_fields"] = np.asarray(REPORT_FIELDS)
    out = os.path.join(HERE, "kats.npz")
    np.savez_compressed(out, **data)
    print(f"wrote {out}: {len(names)} scenarios")


if __name__ == "__main__":
    main()
