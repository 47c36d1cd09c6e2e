"""GPU parity: the CUDA engine (through the C-ABI) against the reference's
golden fixtures and the CPU oracle.  Every comparison is bitwise: f bytes,
IterationReport fields, tau, eligible masks, CSR snapshots, intra-batch
component labelings."""

import numpy as np
import pytest

from golden_io import (STREAM_CASES, csr_digest, kernel_case, load_case, report_tuple)
from oracle import OracleEngine
from paper_2604_06596_b200 import streams
from paper_2604_06596_b200.batch import BatchUpdate
from paper_2604_06596_b200.errors import ValidationError

pytestmark = pytest.mark.gpu

JACOBI_CASES = [c for c in STREAM_CASES if c != "er_gauss_seidel"]


def _engine(num_classes=2):
    from paper_2604_06596_b200.engine import DynamicGraph, LabelState

    return DynamicGraph(0, num_classes=num_classes), LabelState()


def _cfg(case_or_kw):
    from paper_2604_06596_b200.engine import EngineConfig

    if isinstance(case_or_kw, dict):
        return EngineConfig(**case_or_kw)
    c = case_or_kw
    return EngineConfig(delta=c.delta, tau=c.tau, max_iterations=c.max_iterations,
                        component_init=c.component_init, mode=c.mode)


def _reports(rep):
    return rep if isinstance(rep, list) else [rep]


@pytest.mark.parametrize("name", JACOBI_CASES)
def test_engine_matches_reference_golden(gpu_device, name):
    from paper_2604_06596_b200.engine import apply_batch

    case = load_case(name)
    g, lab = _engine(case.num_classes)
    cfg = _cfg(case)
    for t, b in enumerate(case.batches):
        lab, rep = apply_batch(g, lab, b, cfg)
        F = lab.F
        assert F.shape == case.f[t].shape, (name, t)
        assert F.tobytes() == case.f[t].tobytes(), f"{name} batch {t}: f differs " \
            f"(max abs {np.abs(F - case.f[t]).max():.3g})"
        for c, r in enumerate(_reports(rep)):
            assert report_tuple(r) == tuple(case.rep_i[t, c]), f"{name} batch {t} col {c}"
            assert r.max_change == case.rep_mc[t, c]
        if not b.is_empty:
            if case.tau == "auto":
                assert g.last_tau == case.tau_vals[t], f"{name} batch {t}: tau"
            assert np.array_equal(g.eligible(), case.elig[t]), f"{name} batch {t}: eligible"
            csr = g.csr()
            assert csr_digest(csr.indptr, csr.indices, csr.weights, csr.degrees) == case.csr_sha[t], \
                f"{name} batch {t}: CSR"
            if case.component_init and len(b.insert_ids):
                v, p, c = g.intra_labeling()
                assert np.array_equal(np.stack([v, p, c]), case.intra[t]), f"{name} batch {t}: intra"
    g.close()


@pytest.mark.parametrize("seed", range(4))
def test_kernel_plugin_matches_reference_golden(gpu_device, seed):
    from paper_2604_06596_b200 import kernels as K

    k = kernel_case(seed)
    vals = np.empty(len(k["frontier"]))
    deltas = np.empty(len(k["frontier"]))
    K.jacobi_step(k["indptr"], k["indices"], k["weights"], k["gt"], k["f"], k["frontier"], vals,
                  deltas, 1)
    assert vals.tobytes() == k["vals"].tobytes()
    assert deltas.tobytes() == k["deltas"].tobytes()
    f = k["f"].copy()
    elig = k["elig"].copy()
    max_iters = 10_000 if seed != 0 else 5
    it, upd, mc, warn, left = K.jacobi_run(k["indptr"], k["indices"], k["weights"], k["gt"], f,
                                           k["frontier"], elig, 1e-7, max_iters, 1)
    assert [it, upd, warn, len(left)] == list(k["run_out"])
    assert mc == k["run_mc"][0]
    assert f.tobytes() == k["run_f"].tobytes()
    assert np.array_equal(elig, k["run_elig"])
    assert np.array_equal(left, k["run_left"])
    f3 = k["f"].copy()
    d3 = np.empty(len(k["frontier"]))
    K.gauss_seidel_step(k["indptr"], k["indices"], k["weights"], k["gt"], f3, k["frontier"], d3)
    assert f3.tobytes() == k["gs_f"].tobytes()
    assert d3.tobytes() == k["gs_deltas"].tobytes()


def _compare_with_oracle(batches, num_classes=2, **kw):
    from paper_2604_06596_b200.engine import apply_batch

    g, lab = _engine(num_classes)
    cfg = _cfg(dict(kw))
    orc = OracleEngine(num_classes, threads=4)
    for t, b in enumerate(batches):
        lab, rep = apply_batch(g, lab, b, cfg)
        oreps = orc.apply_batch(b, **kw)
        for r, o in zip(_reports(rep), oreps):
            assert report_tuple(r) == report_tuple(o), f"batch {t}"
            assert r.max_change == o.max_change, f"batch {t}"
            assert r.edges_traversed == o.edges_traversed, f"batch {t}"
        F = lab.F
        of, _ = orc.labels()
        assert F.tobytes() == of.tobytes(), f"batch {t}: max abs {np.abs(F - of).max():.3g}"
    tau = orc.last_tau
    g.close()
    return tau


@pytest.mark.parametrize("seed", [0, 1])
def test_engine_vs_oracle_mixed_blob_stream(gpu_device, seed):
    bl = streams.make_blobs(6000, 16, 2, seed)
    e = streams.knn_graph_exact(bl.x, 10)
    gt = streams.stratified_seeds(bl.classes, 0.01, seed)
    s = streams.phased_stream(6000, e, bl.classes, gt, 600, seed, 0.69, 0.01, 0.30, initial_gt=4)
    _compare_with_oracle(s.batches, delta=1e-5)


def test_engine_vs_oracle_ten_class_columns(gpu_device):
    bl = streams.make_blobs(4000, 32, 10, 7)
    e = streams.knn_graph_exact(bl.x, 10)
    gt = streams.stratified_seeds(bl.classes, 0.01, 7)
    s = streams.phased_stream(4000, e, bl.classes, gt, 500, 7, 0.99, 0.01, 0.0, initial_gt=20)
    _compare_with_oracle(s.batches, num_classes=10, delta=1e-4)


def test_engine_vs_oracle_er_heavy_deletes_explicit_tau(gpu_device):
    n = 5000
    e = streams.erdos_renyi_edges(n, 8, 3)
    classes = np.random.default_rng(3).integers(0, 2, n).astype(np.int8)
    gt = streams.stratified_seeds(classes, 0.02, 3)
    s = streams.phased_stream(n, e, classes, gt, 400, 3, 0.6, 0.02, 0.38, initial_gt=4)
    _compare_with_oracle(s.batches, delta=1e-6, tau=0.55)


def test_engine_budget_and_noinit_vs_oracle(gpu_device):
    bl = streams.make_blobs(3000, 8, 2, 11)
    e = streams.knn_graph_exact(bl.x, 6)
    gt = streams.stratified_seeds(bl.classes, 0.02, 11)
    s = streams.phased_stream(3000, e, bl.classes, gt, 300, 11, 0.8, 0.02, 0.18, initial_gt=4)
    _compare_with_oracle(s.batches, delta=1e-7, max_iterations=7, component_init=False)


def test_single_whole_graph_batch_vs_oracle(gpu_device):
    bl = streams.make_blobs(20000, 16, 2, 5)
    e = streams.knn_graph_exact(bl.x, 10, block=2048)
    gt = {int(v): int(bl.classes[v]) for v in streams.stratified_seeds(bl.classes, 0.01, 5)}
    b = streams.single_batch(20000, e, gt)
    _compare_with_oracle([b], delta=1e-4)


def test_validation_errors_leave_state_unchanged(gpu_device):
    from paper_2604_06596_b200.engine import EngineConfig, apply_batch

    g, lab = _engine()
    cfg = EngineConfig(delta=1e-9)
    pre = BatchUpdate.from_records([(0, [], 0), (1, [(1, 0, 1.0)], None), (2, [(2, 1, 1.0)], 1)])
    apply_batch(g, lab, pre, cfg)
    before = lab.f.copy()
    bad = [
        (BatchUpdate.from_records([(3, [(3, 9, 1.0)], None)], deletes=[1]), "edge to unknown vertex 9"),
        (BatchUpdate.from_records(deletes=[1, 1]), "duplicate vertex id in deletes"),
        (BatchUpdate.from_records(deletes=[7]), "unknown vertex id 7 in deletes"),
        (BatchUpdate.from_records([(4, [], None)]), "insert ids must be the contiguous block 3..3"),
        (BatchUpdate.from_records([(3, [(3, 0, -1.0)], None)]), "negative weight on edge to vertex 0"),
        (BatchUpdate.from_records([(3, [(3, 1, 1.0)], None)], deletes=[1]),
         "edge to vertex 1 deleted in the same batch"),
        (BatchUpdate.from_records([(3, [], 2)]), "ground-truth class must be 0 or 1"),
    ]
    for batch, msg in bad:
        with pytest.raises(ValidationError, match=msg):
            apply_batch(g, lab, batch, cfg)
    assert g.num_slots == 3 and g.num_alive == 3 and g.edge_count == 2
    assert np.array_equal(lab.f, before)
    g.close()


def test_bitwise_repeatable(gpu_device):
    from paper_2604_06596_b200.engine import EngineConfig, apply_batch

    bl = streams.make_blobs(5000, 16, 2, 21)
    e = streams.knn_graph_exact(bl.x, 10)
    gt = streams.stratified_seeds(bl.classes, 0.01, 21)
    s = streams.phased_stream(5000, e, bl.classes, gt, 1000, 21, 0.9, 0.01, 0.09, initial_gt=4)
    blobs = set()
    for _ in range(3):
        g, lab = _engine()
        for b in s.batches:
            apply_batch(g, lab, b, EngineConfig(delta=1e-6))
        blobs.add(lab.f.tobytes())
        g.close()
    assert len(blobs) == 1


@pytest.mark.parametrize("ncls,long_row,hub_row", [(10, 8, 24), (2, 12, 30), (10, 0, 0)])
def test_row_class_paths(gpu_device, ncls, long_row, hub_row):
    """The LP kernel's short (multi-row warp tiles), long (single-row warp
    tiles) and hub (CTA-cooperative, double-buffered) paths, forced to mix in
    the same rounds by low thresholds, stay bit-identical to the oracle."""
    import os
    import subprocess
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ, DLP_LONG_ROW=str(long_row), DLP_HUB_ROW=str(hub_row))
    r = subprocess.run([sys.executable, os.path.join(here, "_row_class_check.py"), str(ncls)], env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr


def test_ingestion_pipeline_staging_growth(gpu_device):
    """Staging slots outgrown between pipelined batches (floor 0): bit-identical."""
    import os
    import subprocess
    import sys

    here = os.path.dirname(os.path.abspath(__file__))
    env = dict(os.environ, DLP_STAGE_FLOOR_MB="0")
    r = subprocess.run([sys.executable, os.path.join(here, "_staging_check.py")], env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr


def test_ingestion_pipeline_identical_and_atomic(gpu_device):
    """apply_batch(..., next_batch=) validates and stages the next batch while
    the current one runs: identical reports and labels; a bad next batch is
    reported by its own call and leaves the engine unchanged."""
    from paper_2604_06596_b200.engine import DynamicGraph, EngineConfig, LabelState, apply_batch, run_batches

    bl = streams.make_blobs(3000, 16, 3, 2)
    e = streams.knn_graph_exact(bl.x, 8)
    gt = streams.stratified_seeds(bl.classes, 0.02, 2)
    s = streams.phased_stream(3000, e, bl.classes, gt, 300, 2, 0.8, 0.02, 0.18, initial_gt=6)
    cfg = EngineConfig(delta=1e-5)
    g1, l1 = DynamicGraph(0, num_classes=3), LabelState()
    r1 = run_batches(g1, l1, s.batches, cfg, pipelined=False)
    g2, l2 = DynamicGraph(0, num_classes=3), LabelState()
    r2 = run_batches(g2, l2, s.batches, cfg, pipelined=True)
    for a, b in zip(r1, r2):
        assert [(x.iterations, x.updates, x.max_change) for x in a] == [(x.iterations, x.updates, x.max_change) for x in b]
    assert l1.F.tobytes() == l2.F.tobytes()
    # a next batch that deletes an unknown vertex: the error comes from its own call
    bad = BatchUpdate(t=99, insert_ids=np.empty(0, np.int64), insert_gt=np.empty(0, np.int8),
                      edge_owner=np.empty(0, np.int64), edge_other=np.empty(0, np.int64),
                      edge_w=np.empty(0), deletes=np.array([10 ** 9], np.int64))
    g3, l3 = DynamicGraph(0, num_classes=3), LabelState()
    apply_batch(g3, l3, s.batches[0], cfg, next_batch=bad)
    F_before = l3.F.copy()
    with pytest.raises(ValidationError):
        apply_batch(g3, l3, bad, cfg)
    assert l3.F.tobytes() == F_before.tobytes()
    for g in (g1, g2, g3):
        g.close()


def test_staged_batch_invalidated_by_device_batch(gpu_device):
    """A batch staged by the ingestion pipeline was validated against the host
    mirror of its time; a device batch applied in between must invalidate it,
    so the stale batch is re-validated and rejected (graph.py:267-277)."""
    import torch

    from paper_2604_06596_b200.engine import EngineConfig, apply_batch

    g, lab = _engine()
    cfg = EngineConfig(delta=1e-6)
    b1 = BatchUpdate.from_records([(0, [], 1), (1, [(1, 0, 1.0)], None), (2, [(2, 1, 0.5)], 0)])
    b2 = BatchUpdate.from_records([(3, [(3, 2, 1.0)], None), (4, [(4, 3, 1.0)], None)], t=2)
    apply_batch(g, lab, b1, cfg, next_batch=b2)
    ids = torch.tensor([3], dtype=torch.int64, device="cuda")
    dev = dict(t=1, n_ins=1, n_edges=1, n_del=0, insert_ids=ids,
               insert_gt=torch.tensor([-1], dtype=torch.int8, device="cuda"),
               edge_owner=torch.tensor([0], dtype=torch.int64, device="cuda"),
               edge_other=torch.tensor([2], dtype=torch.int64, device="cuda"),
               edge_w=torch.tensor([1.0], dtype=torch.float64, device="cuda"),
               deletes=torch.empty(0, dtype=torch.int64, device="cuda"))
    g.apply_device(dev, cfg, trusted=True)
    assert g.num_slots == 4
    with pytest.raises(ValidationError, match="insert ids must be the contiguous block 4..5"):
        apply_batch(g, lab, b2, cfg)
    assert g.num_slots == 4
    g.close()


def test_nonfinite_weights_nan_labels_like_oracle(gpu_device):
    """An infinite edge weight drives unlabeled labels to NaN (the reference
    keeps NaN: _csr.pyx:52-56 clamps only ordered values).  Such a NaN is an
    unlabeled label, never a boxed ground-truth word: neighbours propagate it
    exactly like the oracle does."""
    from paper_2604_06596_b200.engine import EngineConfig, apply_batch

    recs = [(0, [], 1), (1, [(1, 0, 1.0)], None), (2, [(2, 1, float("inf"))], None),
            (3, [(3, 2, 1.0)], None), (4, [(4, 3, 2.0)], None), (5, [(5, 0, 1.0)], 0)]
    b = BatchUpdate.from_records(recs)
    g, lab = _engine()
    orc = OracleEngine(2)
    cfg = EngineConfig(delta=1e-6, max_iterations=40)
    lab, rep = apply_batch(g, lab, b, cfg)
    orep = orc.apply_batch(b, delta=1e-6, max_iterations=40)
    assert report_tuple(_reports(rep)[0]) == report_tuple(orep[0])
    f, of = lab.f, orc.labels()[0][0]
    assert np.isnan(of).any()
    assert np.array_equal(np.isnan(f), np.isnan(of))
    assert np.array_equal(f[~np.isnan(f)], of[~np.isnan(of)])
    g.close()


def test_too_many_classes_is_a_validation_error(gpu_device):
    from paper_2604_06596_b200.engine import DynamicGraph

    with pytest.raises(ValidationError, match="num_classes must be <= 16"):
        DynamicGraph(0, num_classes=17)
