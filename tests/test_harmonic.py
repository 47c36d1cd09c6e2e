"""The closed-form oracle on the device: harmonic_solve /
stlp (baselines.py:109-190, 278-318) as a dense Cholesky on the B200.

* against the reference's own harmonic_solve / stlp_solve on the known-answer
  scenarios (tests/golden/kats.npz, made by running the reference);
* the reference's accuracy contract: a converged DynLP batch matches the
  closed form within 1e-6 (test_engine.py:154-162, test_acceptance.py:60-82);
* one-vs-rest linearity on a multi-class stream: the C column solutions of
  every free vertex sum to 1 (the harmonic extension of the constant 1);
* the dense cap and the ground-truth preconditions raise ValidationError.
"""

import numpy as np
import pytest

from paper_2604_06596_b200 import streams
from paper_2604_06596_b200.errors import ValidationError
from test_reference_kats import NAMES, Z, scenario

pytestmark = pytest.mark.gpu


def _replay(name):
    from paper_2604_06596_b200.engine import DynamicGraph, EngineConfig, LabelState, apply_batch

    batches, cfgs, _, _ = scenario(name)
    g, lab = DynamicGraph(0), LabelState()
    for b, kw in zip(batches, cfgs):
        lab, _ = apply_batch(g, lab, b, EngineConfig(**kw))
    return g, lab


@pytest.mark.parametrize("name", NAMES)
def test_harmonic_matches_reference(name, gpu_device):
    from paper_2604_06596_b200.engine import harmonic_solve

    g, lab = _replay(name)
    f, info = harmonic_solve(g, lab, return_info=True)
    want = Z[name + "/harmonic"]
    np.testing.assert_allclose(f, want, atol=1e-10, rtol=0)
    alive = g.alive
    assert info["unreachable_pinned"] >= 0
    st = Z[name + "/stlp"]
    if np.isnan(st).any():
        with pytest.raises(ValidationError, match="both classes"):
            g.harmonic(stlp=True)
    else:
        fs, _ = g.harmonic(stlp=True)
        unl = np.flatnonzero(alive & (lab.gt == -1))
        np.testing.assert_allclose(fs[0][unl], st[unl], atol=1e-10, rtol=0)
    g.close()


def test_converged_dynlp_matches_closed_form(gpu_device):
    """test_acceptance.py:60-82 (c01): DynLP at a tight delta vs the oracle."""
    from paper_2604_06596_b200.engine import (DynamicGraph, EngineConfig, LabelState, apply_batch,
                                               harmonic_solve, oracle_batch_solve)

    bl = streams.make_blobs(1500, 8, 2, 3)
    edges = streams.knn_graph_exact(bl.x, 8)
    gt = streams.stratified_seeds(bl.classes, 0.02, 3)
    s = streams.phased_stream(1500, edges, bl.classes, gt, 300, 3, 0.99, 0.01, 0.0, initial_gt=4)
    g, lab = DynamicGraph(0), LabelState()
    cfg = EngineConfig(delta=1e-10, max_iterations=10_000_000)
    for b in s.batches:
        lab, rep = apply_batch(g, lab, b, cfg)
        assert rep.converged
    f = harmonic_solve(g, lab)
    unl = lab.unlabeled_ids(g)
    np.testing.assert_allclose(lab.f[unl], f[unl], atol=1e-6, rtol=0)
    # oracle_batch_solve on a second engine fed the same stream lands on the closed form
    g2, lab2 = DynamicGraph(0), LabelState()
    for b in s.batches:
        lab2, r2 = oracle_batch_solve(g2, lab2, b, cfg)
        assert r2.method == "oracle" and r2.converged
    np.testing.assert_allclose(lab2.f[unl], f[unl], atol=1e-12, rtol=0)
    g.close()
    g2.close()


def test_one_vs_rest_columns_sum_to_one(gpu_device):
    from paper_2604_06596_b200.engine import DynamicGraph, EngineConfig, LabelState, apply_batch, harmonic_solve

    bl = streams.make_blobs(1200, 8, 4, 5, spread=2.0)
    edges = streams.knn_graph_exact(bl.x, 8)
    gt = streams.stratified_seeds(bl.classes, 0.03, 5)
    s = streams.phased_stream(1200, edges, bl.classes, gt, 200, 5, 0.8, 0.02, 0.18, initial_gt=8)
    g, lab = DynamicGraph(0, num_classes=4), LabelState()
    for b in s.batches:
        lab, _ = apply_batch(g, lab, b, EngineConfig(delta=1e-6))
    F = harmonic_solve(g, lab)
    assert F.shape == (4, g.num_slots)
    free = np.flatnonzero(g.eligible())  # alive, unlabeled, reaches a seed
    assert len(free) > 0
    np.testing.assert_allclose(F[:, free].sum(axis=0), 1.0, atol=1e-9, rtol=0)
    g.close()


def test_dense_cap_and_preconditions(gpu_device):
    from paper_2604_06596_b200.engine import DynamicGraph, EngineConfig, LabelState, apply_batch, harmonic_solve

    g, lab = _replay("single_batch_harmonic")
    with pytest.raises(ValidationError, match="dense-solve cap"):
        harmonic_solve(g, lab, dense_cap=10)
    g.close()
    from paper_2604_06596_b200.batch import BatchUpdate

    g, lab = DynamicGraph(0), LabelState()
    lab, _ = apply_batch(g, lab, BatchUpdate.from_records([(0, [], None), (1, [(1, 0, 1.0)], None)]),
                         EngineConfig())
    with pytest.raises(ValidationError, match="ground-truth"):
        harmonic_solve(g, lab)
    g.close()
