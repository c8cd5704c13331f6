"""Parity of the K10 epilogues (FSRw, pooling,
filter_pooled, embedding) at C1 against the reference's own outputs
(tests/golden/epi.npz from make_golden.py) and, on the device's own
decomposition, against the oracle restatement.

Tolerances: fp64 ("parity mode") scores within 1e-9 relative L2 of the
reference (as test_gpu_parity_c1 for x), pooled orders identical; on the same
decomposition the CSR products are bitwise scipy's (CSR order, separately
rounded fp64) and the BLAS-backed ones within 1e-13.  fp32 within 1e-4.
"""

import numpy as np
import pytest
import scipy.sparse as sp

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import fsr_oracle as O  # noqa: E402
from paper_1703_06935_b200 import ranking, spectral  # noqa: E402
from paper_1703_06935_b200.sparsemat import SparseSymmetricMatrix  # noqa: E402
from paper_1703_06935_b200.workloads import CONFIGS, cluster_descriptors  # noqa: E402

PAIRS = ((0, 1), (2, 3), (4, 4), (5, 9))


def rel_l2(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.fixture(scope="module")
def c1(golden):
    g, e = golden("c1"), golden("epi")
    n, r, p, q, tau, seed = (int(v) for v in g["params"])
    cfg = CONFIGS["C1"]
    data, queries, _ = cluster_descriptors(cfg)
    S = SparseSymmetricMatrix(sp.csr_matrix((g["S_data"], g["W_indices"], g["W_indptr"]), shape=(n, n)))
    P = ranking.PoolingMatrix.from_region_map(e["r2i"], weights=e["pool_w"])
    ys = [ranking.ObservationVector(n, g["y_idx"][g["y_ptr"][j]:g["y_ptr"][j + 1]],
                                    g["y_val"][g["y_ptr"][j]:g["y_ptr"][j + 1]], cap=cfg.y_top)
          for j in range(e["a_fsrw"].shape[0])]
    return g, e, cfg, data, queries, S, P, ys, dict(r=r, p=p, q=q, tau=tau, seed=seed)


@pytest.fixture(scope="module", params=["float64", "float32"])
def decs(request, c1):
    *_, S, P, ys, prm = c1
    dec = spectral.decompose(S, prm["r"], p=prm["p"], q=prm["q"], seed=prm["seed"], dtype=request.param)
    sdec = spectral.sparsify(dec, prm["tau"])
    return request.param, {"a": dec, "s": sdec}


def tol(dtype):
    return 1e-9 if dtype == "float64" else 1e-4


@pytest.mark.parametrize("tag", ["a", "s"])
def test_fsrw_matches_reference(c1, decs, tag):
    g, e, cfg, data, queries, S, P, ys, _ = c1
    dtype, d = decs
    h = ranking.h_alpha(float(g["alpha"]))
    for j, y in enumerate(ys):
        x = ranking.filter(d[tag], h, y)
        xw = ranking.fsrw_correct(x, d[tag], data, queries[j])
        assert rel_l2(xw, e[f"{tag}_fsrw"][j]) < tol(dtype)
        if dtype == "float64":  # same decomposition: only the V q dot order differs
            ref = O.fsrw_correct(x, d[tag].eta, data, queries[j])
            np.testing.assert_allclose(xw, ref, rtol=1e-13, atol=1e-15)


@pytest.mark.parametrize("tag", ["a", "s"])
def test_pooling_matches_reference(c1, decs, tag):
    g, e, cfg, data, queries, S, P, ys, _ = c1
    dtype, d = decs
    h = ranking.h_alpha(float(g["alpha"]))
    Ub = ranking.pooled_basis(P, d[tag])
    # fp32 SPARSE keeps a slightly different support than the fp64 reference
    # (tau-boundary flips): check it against the oracle on the
    # device's own U~ instead of the reference fixture.
    vs_reference = not (dtype == "float32" and tag == "s")
    if vs_reference:
        assert rel_l2(Ub[:200], e[f"{tag}_ubar_head"]) < tol(dtype)
        assert rel_l2(Ub.sum(axis=1), e[f"{tag}_ubar_rowsum"]) < tol(dtype)
    U_host = d[tag].U
    if dtype == "float64":
        np.testing.assert_array_equal(Ub, O.pooled_basis(P.csr, U_host))  # scipy order, bitwise
    else:
        assert rel_l2(Ub, O.pooled_basis(P.csr, U_host)) < 1e-6
    for j, y in enumerate(ys):
        x = ranking.filter(d[tag], h, y)
        xp = ranking.pool(P, x)
        if vs_reference:
            assert rel_l2(xp, e[f"{tag}_pool"][j]) < tol(dtype)
        else:
            assert rel_l2(xp, O.pool(P.csr, x)) < 1e-6
        if dtype == "float64":
            np.testing.assert_array_equal(xp, O.pool(P.csr, x))
            res = ranking.RankingResult.from_scores(x, P)
            np.testing.assert_array_equal(res.order[:100], e[f"{tag}_pooled_order"][j])
        xf = ranking.filter_pooled(d[tag], h, y, Ub)
        if vs_reference:
            assert rel_l2(xf, e[f"{tag}_filter_pooled"][j]) < tol(dtype)
        else:
            w = ranking.transfer_values(h, d[tag].eigenvalues)
            assert rel_l2(xf, O.filter_pooled(U_host, w, y.indices, y.values, Ub)) < 1e-5


@pytest.mark.parametrize("tag", ["a", "s"])
def test_embedding_similarity_matches_reference(c1, decs, tag):
    g, e, cfg, data, queries, *_ = c1
    dtype, d = decs
    h = ranking.h_alpha(float(g["alpha"]))
    phi = ranking.embedding(d[tag], h)
    sims = [ranking.out_of_sample_similarity(queries[a], queries[b], phi, data, cfg.y_top, cfg.gamma)
            for a, b in PAIRS]
    np.testing.assert_allclose(sims, e[f"{tag}_oos"], rtol=tol(dtype) * 10)
    if dtype == "float64":  # the materialised Phi is the reference's object, value for value
        w = ranking.transfer_values(h, d[tag].eigenvalues)
        ref = O.embedding(d[tag].U, w)
        m = phi.matrix()
        if sp.issparse(ref):
            # scipy's product leaves the reference's column indices unsorted: compare canonical forms
            assert sp.issparse(m) and m.shape == ref.shape
            m, ref = m.sorted_indices(), ref.sorted_indices()
            np.testing.assert_array_equal(m.indptr, ref.indptr)
            np.testing.assert_array_equal(m.indices, ref.indices)
            np.testing.assert_allclose(m.data, ref.data, rtol=1e-15)
        else:
            np.testing.assert_allclose(m, ref, rtol=1e-15)


def test_filter_pooled_batch_equals_single(c1, decs):
    g, e, cfg, data, queries, S, P, ys, _ = c1
    dtype, d = decs
    h = ranking.h_alpha(float(g["alpha"]))
    dec = d["s"]
    Ub = ranking.pooled_basis_device(P, dec)
    q = ranking.DeviceQueries(ranking.QueryBatch.from_vectors(ys), dec.dtype, Ub.device)
    Xb = ranking.filter_pooled_device(dec, h, q, Ub).double().cpu().numpy()
    for j, y in enumerate(ys):
        np.testing.assert_allclose(Xb[j], ranking.filter_pooled(dec, h, y, Ub),
                                   rtol=1e-5 if dtype == "float32" else 1e-12, atol=1e-12)


def test_fsrw_batch_equals_single(c1, decs):
    g, e, cfg, data, queries, S, P, ys, _ = c1
    dtype, d = decs
    h = ranking.h_alpha(float(g["alpha"]))
    dec = d["a"]
    X = torch.as_tensor(ranking.filter_batch(dec, h, ys)).to(device="cuda", dtype=dec.dtype)
    V = torch.as_tensor(data).to(device="cuda", dtype=dec.dtype)
    Qs = torch.as_tensor(np.stack([queries[j] for j in range(len(ys))])).to(device="cuda", dtype=dec.dtype)
    ranking.fsrw_correct_device(X, dec, V, Qs)
    for j, y in enumerate(ys):
        single = ranking.fsrw_correct(ranking.filter(dec, h, y), dec, data, queries[j])
        np.testing.assert_allclose(X[j].double().cpu().numpy(), single, rtol=1e-5 if dtype == "float32" else 1e-12,
                                   atol=1e-7 if dtype == "float32" else 1e-15)


def test_epilogue_errors(c1, decs):
    g, e, cfg, data, queries, S, P, ys, _ = c1
    _, d = decs
    with pytest.raises(ValueError):
        ranking.PoolingMatrix(sp.csr_matrix(np.array([[1.0, 1.0], [1.0, 0.0]])))  # region 0 in two images
    with pytest.raises(ValueError):
        ranking.PoolingMatrix(sp.csr_matrix(np.array([[1.0, -1.0]])))
    with pytest.raises(ValueError):
        ranking.pool(P, np.zeros(7))
    with pytest.raises(ValueError):
        ranking.fsrw_correct(np.zeros(5), d["a"], data, queries[0])
    with pytest.raises(ValueError):
        ranking.fsrw_correct(np.zeros(data.shape[0]), d["a"], data, 2.0 * queries[0])
    with pytest.raises(ValueError):
        ranking.pooled_basis(ranking.PoolingMatrix.identity(7), d["a"])
    neg = ranking.custom_transfer(lambda x: x - 2.0, nondecreasing=True)
    with pytest.raises(ValueError):
        ranking.embedding(d["a"], neg)
