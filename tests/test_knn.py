"""k-NN edge construction (builder.py:42-92): the CPU restatement pinned to
the reference's own outputs, and the B200 tensor-core path (screen + exact
fp64 re-check) against both: pair sets exact, weights within 1e-12
(tests/test_builder.py:66 tolerance)."""

import numpy as np
import pytest

from knn_golden import cases
from oracle import knn_oracle

CASES = cases()


@pytest.mark.parametrize("name", sorted(CASES))
def test_oracle_matches_reference_knn(name):
    c = CASES[name]
    u, v, w = knn_oracle.knn_graph(c["x"], c["k"], c["mode"])
    assert np.array_equal(u, c["u"]) and np.array_equal(v, c["v"])
    assert np.allclose(w, c["w"], rtol=0, atol=1e-12)


def test_oracle_validation_messages():
    with pytest.raises(knn_oracle.OracleValidationError, match="row 1"):
        knn_oracle.knn_graph(np.array([[1.0, 0.0], [0.0, 0.0]]), 1)
    with pytest.raises(knn_oracle.OracleValidationError):
        knn_oracle.knn_graph(np.eye(3), 3)


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(CASES))
def test_b200_knn_graph_matches_reference(gpu_device, name):
    from paper_2604_06596_b200.knn import knn_graph

    c = CASES[name]
    e = knn_graph(c["x"], c["k"], similarity_mode=c["mode"])
    assert np.array_equal(e.u, c["u"]) and np.array_equal(e.v, c["v"]), name
    assert np.allclose(e.w, c["w"], rtol=0, atol=1e-12), name


@pytest.mark.gpu
def test_b200_knn_validation(gpu_device):
    from paper_2604_06596_b200.errors import ValidationError
    from paper_2604_06596_b200.knn import knn_graph

    with pytest.raises(ValidationError, match="row 1"):
        knn_graph(np.array([[1.0, 0.0], [0.0, 0.0]]), 1)
    with pytest.raises(ValidationError):
        knn_graph(np.eye(3), 0)
    with pytest.raises(ValidationError):
        knn_graph(np.eye(3), 3)


@pytest.mark.gpu
@pytest.mark.parametrize("n,dim,k,seed", [(20000, 128, 10, 0), (12000, 64, 16, 1), (5000, 16, 10, 2)])
def test_b200_knn_query_rows_exact(gpu_device, n, dim, k, seed):
    """Top-k rows of arriving points against the whole dataset equal the
    fp64 selection by (-sim, id); the tensor-core screen is within its
    error bound of the exact sims."""
    from paper_2604_06596_b200 import streams
    from paper_2604_06596_b200.knn import KnnIndex

    x = streams.make_blobs(n, dim, 10, seed).x
    idx = KnnIndex(x)
    q0, q1 = n // 3, n // 3 + 700
    ids, sims = idx.query(q0, q1, k)
    st = idx.stats()
    xn = x / np.linalg.norm(x, axis=1, keepdims=True)
    s = xn[q0:q1] @ xn.T
    s[np.arange(q1 - q0), np.arange(q0, q1)] = -np.inf
    order = np.lexsort((np.broadcast_to(np.arange(n), s.shape), -s), axis=-1)[:, :k]
    assert np.array_equal(ids, order)
    assert np.allclose(sims, np.take_along_axis(s, order, axis=1), rtol=0, atol=1e-13)
    # screened candidates: within eps of exact, and they contain the true top-k
    ns, val, cid, thr = idx.debug_candidates(q0, q1)
    ok = cid >= 0
    exact = np.einsum("qd,qcd->qc", xn[q0:q1], xn[np.where(ok, cid, 0)])
    assert np.abs(np.where(ok, val - exact, 0)).max() <= st.eps
    assert st.fallback_queries <= (q1 - q0) // 50, st
    idx.close()
