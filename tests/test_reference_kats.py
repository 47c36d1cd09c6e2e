"""The reference's engine-level known-answer tests, restated on the B200 engine.

Fixture: tests/golden/kats.npz (tests/golden/make_kat_golden.py runs the REAL
reference over each scenario).  Every scenario is checked three ways:

* the known answer the reference test asserts (test_engine.py line cited per
  scenario), on the B200 engine's labels and report;
* bitwise against the reference's own run of the same stream (f bytes and
  every IterationReport field, max_change included);
* the closed-form harmonic labels (baselines.harmonic_solve) within the
  reference test's 1e-6 where the reference test compares them.

The CPU test pins the C oracle to the same fixture.
"""

import os

import numpy as np
import pytest

from oracle import OracleEngine
from paper_2604_06596_b200.batch import BatchUpdate

HERE = os.path.dirname(os.path.abspath(__file__))
Z = np.load(os.path.join(HERE, "golden", "kats.npz"))
NAMES = [str(x) for x in Z["names"]]
FIELDS = [str(x) for x in Z["report_fields"]]


def scenario(name):
    p = name + "/"
    io, eo, do = Z[p + "io"], Z[p + "eo"], Z[p + "do"]
    batches, cfgs = [], []
    for t in range(len(io) - 1):
        c = Z[p + "cfg"][t]
        batches.append(BatchUpdate(t=int(c[3]), insert_ids=Z[p + "ids"][io[t]:io[t + 1]].astype(np.int64),
                                   insert_gt=Z[p + "gt"][io[t]:io[t + 1]].astype(np.int8),
                                   edge_owner=Z[p + "own"][eo[t]:eo[t + 1]].astype(np.int64),
                                   edge_other=Z[p + "oth"][eo[t]:eo[t + 1]].astype(np.int64),
                                   edge_w=Z[p + "w"][eo[t]:eo[t + 1]].astype(np.float64),
                                   deletes=Z[p + "dels"][do[t]:do[t + 1]].astype(np.int64)))
        cfgs.append(dict(delta=float(c[0]), tau="auto" if np.isnan(c[1]) else float(c[1]),
                         max_iterations=None if c[2] < 0 else int(c[2])))
    fn = Z[p + "f_n"]
    fo = np.concatenate([[0], np.cumsum(fn)])
    fs = [Z[p + "f"][fo[t]:fo[t + 1]] for t in range(len(fn))]
    return batches, cfgs, Z[p + "reports"], fs


def check_known_answer(name, f, reps, gt, alive, harmonic):
    """The assertion of the reference test the scenario restates."""
    last = reps[-1]
    if name == "empty_batch":  # test_engine.py:131-140
        assert last["iterations"] == 0 and last["converged"]
    elif name == "structural_trace":  # test_engine.py:186-192
        assert last["iterations"] >= 2 and last["converged"]
        assert f[7] < 0.5 < f[9]
    elif name == "new_gt_seed":  # test_engine.py:205-208
        assert f[3] == 1.0 and f[1] > 0.5 and last["iterations"] >= 1
    elif name == "delete_gt":  # test_engine.py:215-218
        assert abs(f[1] - 0.5) <= 1e-8
    elif name == "unreachable_pin":  # test_engine.py:236-238
        assert f[1] == 0.5 and last["isolated_pinned"] == 1
    elif name == "budget_two":  # test_engine.py:246-248
        assert not last["converged"] and last["iterations"] == 2
    elif name.startswith("fixed_point"):  # test_engine.py:258-262 (residual <= delta)
        assert last["converged"]
    if name in ("structural_trace", "single_batch_harmonic"):  # test_engine.py:159-162, 190-192
        unl = np.flatnonzero(alive.astype(bool) & (gt == -1))
        np.testing.assert_allclose(f[unl], harmonic[unl], atol=1e-6, rtol=0)


def rep_dict(r):
    return {k: (bool(getattr(r, k)) if k == "converged" else getattr(r, k)) for k in FIELDS}


def ref_dict(row):
    return {k: (bool(v) if k == "converged" else v) for k, v in zip(FIELDS, row)}


def test_kat_fixture_known_answers():
    """The fixture itself satisfies the reference tests' assertions."""
    for name in NAMES:
        _, _, reps, fs = scenario(name)
        p = name + "/"
        check_known_answer(name, fs[-1], [ref_dict(r) for r in reps], Z[p + "gt_final"], Z[p + "alive"],
                           Z[p + "harmonic"])


@pytest.mark.parametrize("name", NAMES)
def test_oracle_matches_reference_kats(name):
    batches, cfgs, reps, fs = scenario(name)
    orc = OracleEngine(2)
    for t, (b, kw) in enumerate(zip(batches, cfgs)):
        o = orc.apply_batch(b, **kw)[0]
        assert (o.iterations, o.updates, o.max_change, bool(o.converged)) == \
            (reps[t][0], reps[t][1], reps[t][2], bool(reps[t][3])), (name, t)
        f, _ = orc.labels()
        assert f.reshape(-1)[:len(fs[t])].tobytes() == fs[t].tobytes(), (name, t)


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_engine_known_answers_bitwise(name, gpu_device):
    from paper_2604_06596_b200.engine import DynamicGraph, EngineConfig, LabelState, apply_batch

    batches, cfgs, reps, fs = scenario(name)
    g, lab = DynamicGraph(0), LabelState()
    mine = []
    for t, (b, kw) in enumerate(zip(batches, cfgs)):
        lab, r = apply_batch(g, lab, b, EngineConfig(**kw))
        mine.append(rep_dict(r))
        assert mine[-1] == ref_dict(reps[t]), (name, t, mine[-1], reps[t])
        assert lab.f.tobytes() == fs[t].tobytes(), (name, t)
    p = name + "/"
    check_known_answer(name, lab.f, mine, lab.gt, g.alive.astype(np.uint8), Z[p + "harmonic"])
    g.close()


# ---------------------------------------------------------------------------
# The reference's kernel tests (tests/test_kernels.py) against the b200 plugin
# backend (paper_2604_06596_b200.kernels, the DYNLP_KERNELS=b200 module of
# INTEGRATION.md §1), on the reference's own random_state instances.  The
# reference asserts 1e-14 / 1e-12 agreement across backends; this checks bytes.
# ---------------------------------------------------------------------------
def kern(seed):
    p = f"kern{seed}/"
    return {k[len(p):]: Z[k] for k in Z.files if k.startswith(p)}


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(5))
def test_plugin_jacobi_step_matches_reference(seed, gpu_device):  # test_kernels.py:34-44
    from paper_2604_06596_b200 import kernels as kb

    k = kern(seed)
    f = k["f"].copy()
    vals, deltas = np.empty(len(k["unl"])), np.empty(len(k["unl"]))
    kb.jacobi_step(k["indptr"], k["indices"], k["weights"], k["gt"], f, k["unl"], vals, deltas, 1)
    assert vals.tobytes() == k["step_vals"].tobytes()
    assert deltas.tobytes() == k["step_deltas"].tobytes()
    assert f.tobytes() == k["f"].tobytes()  # test_kernels.py:80-85 jacobi_step does not commit


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(5))
def test_plugin_jacobi_run_matches_reference(seed, gpu_device):  # test_kernels.py:46-61
    from paper_2604_06596_b200 import kernels as kb

    k = kern(seed)
    f, elig = k["f"].copy(), k["eligible"].copy()
    it, upd, mc, warn, left = kb.jacobi_run(k["indptr"], k["indices"], k["weights"], k["gt"], f, k["unl"], elig,
                                            1e-6, 10_000, 1)
    assert [it, upd, mc, warn, len(left)] == list(k["run_out"])
    assert f.tobytes() == k["run_f"].tobytes()
    assert elig.tobytes() == k["run_elig"].tobytes()


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(3))
def test_plugin_gauss_seidel_matches_reference(seed, gpu_device):  # test_kernels.py:63-77
    from paper_2604_06596_b200 import kernels as kb

    k = kern(seed)
    f = k["f"].copy()
    d = np.empty(len(k["unl"]))
    kb.gauss_seidel_step(k["indptr"], k["indices"], k["weights"], k["gt"], f, k["unl"], d)
    assert f.tobytes() == k["gs_f"].tobytes()
    assert d.tobytes() == k["gs_deltas"].tobytes()


@pytest.mark.gpu
def test_plugin_contracts(gpu_device):  # test_kernels.py:87-112
    from paper_2604_06596_b200 import kernels as kb

    # isolated vertex sentinel: graph 0-1, vertex 2 isolated with f = 0.9
    indptr = np.array([0, 1, 2, 2], np.int64)
    indices = np.array([1, 0], np.int64)
    weights = np.array([1.0, 1.0])
    gt = np.full(3, -1, np.int8)
    f = np.array([0.5, 0.5, 0.9])
    vals, deltas = np.empty(1), np.empty(1)
    kb.jacobi_step(indptr, indices, weights, gt, f, np.array([2], np.int64), vals, deltas, 1)
    assert vals[0] == 0.5 and deltas[0] == -1.0
    # Gauss-Seidel reads fresh values: chain 0-1-2, 0 labelled 1
    indptr = np.array([0, 1, 3, 4], np.int64)
    indices = np.array([1, 0, 2, 1], np.int64)
    weights = np.ones(4)
    gt = np.array([1, -1, -1], np.int8)
    f = np.array([1.0, 0.0, 0.0])
    d = np.empty(2)
    kb.gauss_seidel_step(indptr, indices, weights, gt, f, np.array([1, 2], np.int64), d)
    assert f[1] == 0.5 and f[2] == 0.5
