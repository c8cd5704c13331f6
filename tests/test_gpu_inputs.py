"""Parity of the device input builders with the
reference: the C1 mutual k-NN graph and observation vectors that
``tests/golden/make_golden.py`` produced with ``specrank.graph`` /
``specrank.ranking``, plus multi-region pooling against the oracle.

Tolerances: graph pattern and query supports identical; weights/values to
1e-12 relative (the device sums each dot product in a different order than
the host BLAS, so the last bits may differ).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import fsr_oracle as O  # noqa: E402
from paper_1703_06935_b200 import knn  # noqa: E402
from paper_1703_06935_b200.workloads import CONFIGS, cluster_descriptors  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def c1_data():
    cfg = CONFIGS["C1"]
    data, queries, _ = cluster_descriptors(cfg)
    return cfg, data, queries


def test_c1_graph_matches_reference(golden, c1_data):
    cfg, data, _ = c1_data
    g = golden("c1")
    W = knn.mutual_knn_graph_device(torch.as_tensor(data).cuda(), cfg.k, cfg.gamma).csr
    np.testing.assert_array_equal(W.indptr, g["W_indptr"])
    np.testing.assert_array_equal(W.indices, g["W_indices"])
    np.testing.assert_allclose(W.data, g["W_data"], rtol=1e-12, atol=0)


def test_c1_graph_bf16_candidates(golden, c1_data):
    """Certified bf16 candidate GEMM + fp64 re-score (the C3 input mode) on C1:
    the reference's graph; every row settled by one of the three stages."""
    cfg, data, _ = c1_data
    g = golden("c1")
    st = {}
    W = knn.mutual_knn_graph_device(torch.as_tensor(data).cuda(), cfg.k, cfg.gamma,
                                    gemm_dtype=torch.bfloat16, stats=st).csr
    assert sum(st.values()) == cfg.n
    np.testing.assert_array_equal(W.indptr, g["W_indptr"])
    np.testing.assert_array_equal(W.indices, g["W_indices"])
    np.testing.assert_allclose(W.data, g["W_data"], rtol=1e-12, atol=0)


def test_c1_observation_vectors_bf16_certified(golden, c1_data):
    """Certified bf16 candidates for the query neighbours: the reference's y."""
    cfg, data, queries = c1_data
    g = golden("c1")
    st = {}
    y_ptr, y_idx, y_val = knn.observation_batch_device(torch.as_tensor(queries).cuda(), torch.as_tensor(data).cuda(),
                                                       cfg.y_top, cfg.gamma, gemm_dtype=torch.bfloat16, stats=st)
    assert sum(st.values()) == len(queries)
    np.testing.assert_array_equal(y_ptr, g["y_ptr"])
    np.testing.assert_array_equal(y_idx, g["y_idx"])
    np.testing.assert_allclose(y_val, g["y_val"], rtol=1e-12, atol=0)


def test_score_error_bound_holds_on_adversarial_rows():
    """The bf16 / bf16x3 candidate-score bounds cover the measured errors of
    the GEMMs they model (rows built to maximise rounding: values just past
    bf16 midpoints, all of one sign)."""
    g = torch.Generator(device="cuda").manual_seed(5)
    for d in (128, 512, 2048):
        A = torch.rand(64, d, generator=g, device="cuda", dtype=torch.float64)
        A = (A.to(torch.bfloat16).double() * (1 + 2.0 ** -9 * 0.999))  # each value ~half a bf16 ulp off
        A /= A.norm(dim=1, keepdim=True)
        X = torch.rand(4096, d, generator=g, device="cuda", dtype=torch.float64)
        X /= X.norm(dim=1, keepdim=True)
        exact = A @ X.T
        for scheme in ("bf16", "bf16x3"):
            err = (knn._approx_sims(A, X, scheme).double() - exact).abs().max().item()
            assert err <= knn.score_error_bound(d, scheme), (d, scheme, err)


def test_c1_observation_vectors_match_reference(golden, c1_data):
    cfg, data, queries = c1_data
    g = golden("c1")
    X = torch.as_tensor(data).cuda()
    Qv = torch.as_tensor(queries).cuda()
    y_ptr, y_idx, y_val = knn.observation_batch_device(Qv, X, cfg.y_top, cfg.gamma)
    np.testing.assert_array_equal(y_ptr, g["y_ptr"])
    np.testing.assert_array_equal(y_idx, g["y_idx"])
    np.testing.assert_allclose(y_val, g["y_val"], rtol=1e-12, atol=0)


@pytest.mark.parametrize("regions,cap", [(3, None), (5, 12), (2, 40)])
def test_pooled_observation_vectors_vs_oracle(regions, cap):
    rng = np.random.default_rng(regions * 100 + (cap or 0))
    n, d, b, k, gamma = 3000, 48, 9, 20, 3.0
    data = rng.standard_normal((n, d))
    data /= np.linalg.norm(data, axis=1, keepdims=True)
    data[7] = data[3]  # exact duplicate: a tie the stable rule must break toward index 3
    reg = rng.standard_normal((b * regions, d))
    reg /= np.linalg.norm(reg, axis=1, keepdims=True)
    y_ptr, y_idx, y_val = knn.observation_batch_device(torch.as_tensor(reg).cuda(), torch.as_tensor(data).cuda(),
                                                       k, gamma, cap=cap, regions=regions)
    for j in range(b):
        oi, ov = O.observation_vector(reg[j * regions:(j + 1) * regions], data, k, gamma, cap=cap)
        s, e = y_ptr[j], y_ptr[j + 1]
        np.testing.assert_array_equal(y_idx[s:e], oi)
        np.testing.assert_allclose(y_val[s:e], ov, rtol=1e-12, atol=0)


def test_graph_ties_and_isolated_vs_oracle():
    """Duplicated vectors (exact ties) and vectors with no positive similarity."""
    rng = np.random.default_rng(5)
    n, d = 600, 16
    data = rng.standard_normal((n, d))
    data[:, 0] = np.abs(data[:, 0]) + 0.5  # mostly positive dots
    data[10:20] = data[5]                  # ten exact duplicates of row 5
    data[50, :] = 0.0
    data[50, 1] = -1.0
    data[51, :] = 0.0
    data[51, 2] = 1.0
    data /= np.linalg.norm(data, axis=1, keepdims=True)
    for k in (1, 4, 15):
        ref = O.mutual_knn_graph(data, k, 2.0)
        W = knn.mutual_knn_graph_device(torch.as_tensor(data).cuda(), k, 2.0).csr
        np.testing.assert_array_equal(W.indptr, ref.indptr)
        np.testing.assert_array_equal(W.indices, ref.indices)
        np.testing.assert_allclose(W.data, ref.data, rtol=1e-12, atol=0)


def test_builders_reject_bad_arguments():
    X = torch.eye(4, dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError):
        knn.mutual_knn_graph_device(X, 4, 3.0)
    with pytest.raises(ValueError):
        knn.mutual_knn_graph_device(X, 0, 3.0)
    with pytest.raises(ValueError):
        knn.mutual_knn_graph_device(X, 2, 0.0)
    with pytest.raises(ValueError):
        knn.observation_batch_device(X, X, 5, 3.0)
    with pytest.raises(ValueError):
        knn.observation_batch_device(X, X, 2, 3.0, cap=0)
