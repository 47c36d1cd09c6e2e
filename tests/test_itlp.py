"""ItLP (baselines.itlp_batch_solve, baselines.py:236-253) on the B200 against
the real reference's outputs (tests/golden/itlp_reference.npz, made by
make_itlp_golden.py): labels bitwise, report fields exact."""

import os

import numpy as np
import pytest

from paper_2604_06596_b200.batch import BatchUpdate

PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "itlp_reference.npz")
Z = np.load(PATH)
NAMES = sorted({k.split("__")[0] for k in Z.files})


def _case(name):
    g = lambda k: Z[f"{name}__{k}"]  # noqa: E731
    io, eo, do = g("b_ins_off"), g("b_edge_off"), g("b_del_off")
    batches = [BatchUpdate(t=int(g("b_t")[t]), insert_ids=g("b_ins")[io[t]:io[t + 1]],
                           insert_gt=g("b_gt")[io[t]:io[t + 1]], edge_owner=g("b_owner")[eo[t]:eo[t + 1]],
                           edge_other=g("b_other")[eo[t]:eo[t + 1]], edge_w=g("b_w")[eo[t]:eo[t + 1]],
                           deletes=g("b_del")[do[t]:do[t + 1]]) for t in range(len(g("b_t")))]
    ncls, delta, mi = g("meta")
    fo = g("f_off")
    fs = [g("f")[fo[t]:fo[t + 1]] for t in range(len(batches))]
    return batches, int(ncls), float(delta), None if mi < 0 else int(mi), fs, g("reps")


def test_itlp_golden_loads():
    for n in NAMES:
        batches, ncls, delta, mi, fs, reps = _case(n)
        assert len(batches) == len(fs) == reps.shape[0]


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_itlp_matches_reference(gpu_device, name):
    from paper_2604_06596_b200.engine import DynamicGraph, EngineConfig, LabelState, itlp_batch_solve

    batches, ncls, delta, mi, fs, reps = _case(name)
    g, lab = DynamicGraph(0, num_classes=ncls), LabelState()
    cfg = EngineConfig(delta=delta, max_iterations=mi)
    for t, b in enumerate(batches):
        lab, rep = itlp_batch_solve(g, lab, b, cfg)
        rr = rep if isinstance(rep, list) else [rep]
        for c, r in enumerate(rr):
            want = reps[t, c]
            got = (r.iterations, r.updates, int(r.converged), r.warnings, r.isolated_pinned, r.unreachable_pinned)
            assert got == tuple(int(x) for x in want[:6]), f"{name} batch {t} col {c}: {got} vs {want}"
            assert r.max_change == want[6], f"{name} batch {t} col {c}"
        F = lab.F
        assert F.tobytes() == fs[t].tobytes(), f"{name} batch {t}: max abs {np.abs(F.ravel() - fs[t]).max():.3g}"
    g.close()
