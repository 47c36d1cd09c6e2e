"""Pin the CPU oracle (oracle/dynlp_oracle.c) against the reference's outputs.

The fixtures in tests/golden/ were produced by running the unmodified
reference (tests/golden/make_golden.py); every comparison here is bitwise.
When the reference itself is importable (this container, or oracle/_ref on
the GPU box) the oracle is additionally run side by side with it on fresh
streams.
"""

import numpy as np
import pytest

from golden_io import (STREAM_CASES, csr_digest, kernel_case, load_case, pairwise_inputs,
                       report_tuple)
from oracle import (OracleEngine, load_reference, orc_gauss_seidel_step, orc_jacobi_run,
                    orc_jacobi_step, pairwise_sum)
from paper_2604_06596_b200 import streams


@pytest.mark.parametrize("name", STREAM_CASES)
def test_oracle_matches_reference_stream(name):
    case = load_case(name)
    orc = OracleEngine(case.num_classes, threads=1)
    for t, b in enumerate(case.batches):
        reps = orc.apply_batch(b, delta=case.delta, tau=case.tau,
                               max_iterations=case.max_iterations,
                               component_init=case.component_init, mode=case.mode)
        f, gt = orc.labels()
        assert f.shape == case.f[t].shape
        assert f.tobytes() == case.f[t].tobytes(), f"{name} batch {t}: f differs"
        for c, r in enumerate(reps):
            assert report_tuple(r) == tuple(case.rep_i[t, c]), f"{name} batch {t} col {c}"
            assert r.max_change == case.rep_mc[t, c]
        if not b.is_empty:
            assert orc.last_tau == case.tau_vals[t] or (case.tau != "auto")
            assert np.array_equal(orc.eligible(), case.elig[t])
            assert csr_digest(*orc.csr()) == case.csr_sha[t], f"{name} batch {t}: CSR"
            if case.component_init and len(b.insert_ids):
                v, p, c = orc.intra_labeling()
                assert np.array_equal(np.stack([v, p, c]), case.intra[t])
    indptr, indices, weights, degrees = orc.csr()
    assert np.array_equal(indptr, case.final[0])
    assert np.array_equal(indices, case.final[1])
    assert weights.tobytes() == case.final[2].tobytes()


def test_pairwise_sum_matches_numpy_mean():
    for a, mean in pairwise_inputs():
        if len(a) == 0:
            continue
        assert pairwise_sum(a) / len(a) == mean, len(a)
        assert float(np.mean(a)) == mean


@pytest.mark.parametrize("seed", range(4))
def test_oracle_kernel_plugin_functions(seed):
    k = kernel_case(seed)
    vals = np.empty(len(k["frontier"]))
    deltas = np.empty(len(k["frontier"]))
    orc_jacobi_step(k["indptr"], k["indices"], k["weights"], k["gt"], k["f"], k["frontier"],
                    vals, deltas, 1)
    assert vals.tobytes() == k["vals"].tobytes()
    assert deltas.tobytes() == k["deltas"].tobytes()
    f = k["f"].copy()
    elig = k["elig"].copy()
    max_iters = 10_000 if seed != 0 else 5
    it, upd, mc, warn, left = orc_jacobi_run(k["indptr"], k["indices"], k["weights"], k["gt"], f,
                                             k["frontier"], elig, 1e-7, max_iters, 1)
    assert [it, upd, warn, len(left)] == list(k["run_out"])
    assert mc == k["run_mc"][0]
    assert f.tobytes() == k["run_f"].tobytes()
    assert np.array_equal(elig, k["run_elig"])
    assert np.array_equal(np.sort(left), k["run_left"])
    f3 = k["f"].copy()
    d3 = np.empty(len(k["frontier"]))
    orc_gauss_seidel_step(k["indptr"], k["indices"], k["weights"], k["gt"], f3, k["frontier"], d3)
    assert f3.tobytes() == k["gs_f"].tobytes()
    assert d3.tobytes() == k["gs_deltas"].tobytes()


def test_oracle_thread_count_bitwise_identical():
    bl = streams.make_blobs(1500, 8, 2, 5)
    e = streams.knn_graph_exact(bl.x, 8)
    gt = streams.stratified_seeds(bl.classes, 0.02, 5)
    s = streams.phased_stream(1500, e, bl.classes, gt, 400, 5, 0.9, 0.02, 0.08, initial_gt=4)
    outs = []
    for threads in (1, 4):
        orc = OracleEngine(2, threads=threads)
        reps = [orc.apply_batch(b, delta=1e-6)[0] for b in s.batches]
        outs.append((orc.labels()[0].tobytes(), [report_tuple(r) for r in reps]))
    assert outs[0] == outs[1]


def _live_reference():
    ref = load_reference()
    if ref is None:
        pytest.skip("reference not importable here")
    return ref


@pytest.mark.parametrize("seed", [0, 1])
def test_oracle_vs_live_reference_mixed_blobs(seed):
    _live_reference()
    from dynlp.engine import EngineConfig, apply_batch
    from dynlp.graph import BatchUpdate as RB
    from dynlp.graph import DynamicGraph
    from dynlp.labels import LabelState

    bl = streams.make_blobs(800, 12, 2, seed + 10)
    e = streams.knn_graph_exact(bl.x, 7)
    gt = streams.stratified_seeds(bl.classes, 0.03, seed)
    s = streams.phased_stream(800, e, bl.classes, gt, 90, seed, 0.65, 0.03, 0.32, initial_gt=4)
    g, lab = DynamicGraph(), LabelState()
    orc = OracleEngine(2)
    cfg = EngineConfig(delta=1e-5, threads=1)
    for b in s.batches:
        rb = RB(b.t, b.insert_ids, b.insert_gt, b.edge_owner, b.edge_other, b.edge_w, b.deletes)
        lab, r = apply_batch(g, lab, rb, cfg)
        (o,) = orc.apply_batch(b, delta=1e-5)
        assert report_tuple(o) == report_tuple(r) and o.max_change == r.max_change
        assert orc.labels()[0][0].tobytes() == lab.f[: g.num_slots].tobytes()


def test_column_parallel_oracle_is_bitwise_serial():
    """The oracle runs one-vs-rest columns concurrently when threads > 1
    (the columns are independent reference runs): identical to serial."""
    from test_long_stream import _stream

    batches = _stream(n_boot=6, n_mixed=8, bs=300, classes=5, seed=3)
    a, b = OracleEngine(5, threads=1), OracleEngine(5, threads=4)
    for t, x in enumerate(batches):
        ra, rb = a.apply_batch(x), b.apply_batch(x)
        assert [(r.iterations, r.updates, r.max_change, r.edges_traversed) for r in ra] == \
            [(r.iterations, r.updates, r.max_change, r.edges_traversed) for r in rb], t
        assert a.labels()[0].tobytes() == b.labels()[0].tobytes(), t


def test_c5_grid3d_knn_exact():
    """C5's generator: exact 3-D Euclidean k-NN of uniform
    cube points, union-symmetrised with max-merge, against brute force."""
    import numpy as np

    from paper_2604_06596_b200 import streams

    b = streams.uniform_cube(3000, 2)
    e = streams.knn_graph_grid3d(b.x, 10)
    d2 = ((b.x[:, None, :] - b.x[None, :, :]) ** 2).sum(-1)
    np.fill_diagonal(d2, np.inf)
    nn = np.argsort(d2, axis=1, kind="stable")[:, :10]
    pairs = set()
    for i in range(len(b.x)):
        for j in nn[i]:
            pairs.add((min(i, int(j)), max(i, int(j))))
    got = set(zip(e.u.tolist(), e.v.tolist()))
    assert got == pairs
    assert (e.w > 0).all() and (e.w <= 1).all()
    assert set(np.unique(b.classes).tolist()) <= {0, 1}
