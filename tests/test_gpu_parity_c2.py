"""End-to-end parity at the FULL BASELINE C2 size against the reference's own
outputs (tests/golden/c2.npz, made by ``make_golden.py c2`` from
/root/reference: n = 1e5, d = 512, 1000 Zipf clusters, mutual kNN k = 50,
gamma = 3, r = 2000, p = 200, q = 3, tau = 5% = 1e7, 1000 queries with
top-50 observation vectors, h_alpha(0.99)).

The fixture holds outputs only; the graph is rebuilt here from the seeded
descriptors with the fp64 device builder and pinned to the reference's by
the sha256 of its (indptr, indices) pattern and a digest of its weights.

Contract (BASELINE.json north_star; reference spectral.py:297-309, :269-294,
ranking.py:229-255, :390-395), asserted PER QUERY where it applies:
  * fp64 parity mode: Ritz values <= 1e-10 normwise; sparse support sha256
    identical; x <= 1e-9 relative L2 (APPROX and SPARSE); top-100 overlap
    >= 0.99 for every one of the 1000 queries (APPROX and SPARSE).
  * fp32: Ritz <= 1e-5 normwise; APPROX x <= 1e-4 and top-100 overlap >= 0.99
    for every query; SPARSE support-aligned (the reference's kept set -- the
    fp64 support, itself pinned by hash -- with the fp32 values) x <= 1e-4;
    SPARSE end-to-end (own top-tau) overlap: mean >= 0.99, per-query minimum
    reported (tau-boundary flips put it at ~0.99).
Set FSR_PARITY_OUT=<file> to write the measured numbers as JSON.
"""

import hashlib
import json
import os
from types import SimpleNamespace

import numpy as np
import pytest
import scipy.sparse as sp

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1703_06935_b200 import graph, knn, ranking, spectral  # noqa: E402
from paper_1703_06935_b200.workloads import CONFIGS, cluster_descriptors  # noqa: E402

RESULTS = {}


def rel_l2(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def overlap(a, b):
    return len(set(np.asarray(a).tolist()) & set(np.asarray(b).tolist())) / len(b)


def weight_digest(data):
    c = np.random.default_rng(99).random(data.size)
    return np.array([data.sum(), np.dot(data, data), np.dot(data, c), data.max() if data.size else 0.0])


def pattern_hash(indptr, indices):
    h = hashlib.sha256(np.ascontiguousarray(indptr, dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(indices, dtype=np.int32).tobytes())
    return h.hexdigest()


def support_hash(U, r):
    coo = U.tocoo()
    flat = np.sort(coo.row.astype(np.int64) * r + coo.col.astype(np.int64))
    return hashlib.sha256(flat.tobytes()).hexdigest()


def record(key, value):
    RESULTS[key] = value
    out = os.environ.get("FSR_PARITY_OUT")
    if out:
        with open(out, "w") as f:
            json.dump(RESULTS, f, indent=1, default=float)


@pytest.fixture(scope="module")
def c2(golden):
    g = golden("c2")
    cfg = CONFIGS["C2"]
    n, r, p, q, tau, seed = (int(v) for v in g["params"])
    assert (n, r, p, q, tau) == (cfg.n, cfg.r, cfg.p, cfg.q, cfg.tau)
    data, qv, _ = cluster_descriptors(cfg)
    X = torch.as_tensor(data).cuda()
    W = knn.mutual_knn_graph_device(X, cfg.k, cfg.gamma)  # fp64 parity builder
    Q = torch.as_tensor(qv).cuda()
    y_ptr, y_idx, y_val = knn.observation_batch_device(Q, X, cfg.y_top, cfg.gamma)
    del X, Q
    S = graph.normalize_adjacency(W, graph.degrees(W))
    batch = ranking.QueryBatch(n, g["y_ptr"], g["y_idx"], g["y_val"])
    return SimpleNamespace(g=g, cfg=cfg, W=W, S=S, batch=batch, P=dict(n=n, r=r, p=p, q=q, tau=tau, seed=seed),
                           y=(y_ptr, y_idx, y_val), h=ranking.h_alpha(float(g["alpha"])))


def test_c2_graph_and_queries_match_reference(c2):
    g = c2.g
    Wc = c2.W.csr
    assert Wc.nnz == int(g["W_nnz"])
    assert pattern_hash(Wc.indptr, Wc.indices) == str(g["W_pattern_hash"])
    np.testing.assert_allclose(weight_digest(Wc.data), g["W_digest"], rtol=1e-12)
    np.testing.assert_allclose(weight_digest(c2.S.csr.data), g["S_digest"], rtol=1e-12)
    y_ptr, y_idx, y_val = c2.y
    np.testing.assert_array_equal(y_ptr, g["y_ptr"])
    np.testing.assert_array_equal(y_idx, g["y_idx"])
    np.testing.assert_allclose(y_val, g["y_val"], rtol=1e-12, atol=0)


def test_c2_graph_from_certified_bf16_candidates(c2):
    """The C3/C4 input mode at the full C2 size: bf16 candidates (certified,
    knn.certified_topk) + fp64 re-score give the reference's graph exactly."""
    from paper_1703_06935_b200.workloads import cluster_descriptors as cd

    g = c2.g
    data, _, _ = cd(c2.cfg)
    st = {}
    W = knn.mutual_knn_graph_device(torch.as_tensor(data).cuda(), c2.cfg.k, c2.cfg.gamma,
                                    gemm_dtype=torch.bfloat16, stats=st).csr
    record("knn_bf16_certification_rows", st)
    assert sum(st.values()) == c2.cfg.n
    assert pattern_hash(W.indptr, W.indices) == str(g["W_pattern_hash"])
    np.testing.assert_allclose(weight_digest(W.data), g["W_digest"], rtol=1e-12)


@pytest.fixture(scope="module", params=["float64", "float32"])
def decs(request, c2):
    P = c2.P
    dec = spectral.decompose(c2.S, P["r"], p=P["p"], q=P["q"], seed=P["seed"], dtype=request.param)
    return request.param, dec, spectral.sparsify(dec, P["tau"])


def topk_all(dec, c2, k=100):
    return ranking.filter_batch(dec, c2.h, c2.batch, topk=k)


def first_queries(c2, m):
    b = c2.batch
    e = int(b.y_ptr[m])
    return ranking.QueryBatch(b.size, b.y_ptr[:m + 1], b.y_idx[:e], b.y_val[:e])


def test_c2_ritz_and_eta(c2, decs):
    g = c2.g
    dtype, dec, sdec = decs
    err = float(np.abs(dec.eigenvalues - g["lam"]).max() / np.abs(g["lam"]).max())
    record(f"{dtype}_ritz_normwise", err)
    assert err <= (1e-10 if dtype == "float64" else 1e-5), err
    assert np.abs(dec.eta - g["eta"]).max() < (1e-8 if dtype == "float64" else 1e-4)


def test_c2_approx_ranking_per_query(c2, decs):
    g = c2.g
    dtype, dec, _ = decs
    nx = g["x_approx"].shape[0]
    X = ranking.filter_batch(dec, c2.h, first_queries(c2, nx))
    errs = [rel_l2(X[j], g["x_approx"][j]) for j in range(nx)]
    record(f"{dtype}_approx_x_rel_l2_max", max(errs))
    assert max(errs) <= (1e-9 if dtype == "float64" else 1e-4), errs
    idx, _ = topk_all(dec, c2)
    ov = np.array([overlap(idx[j], g["top_approx"][j]) for j in range(c2.batch.b)])
    record(f"{dtype}_approx_top100_overlap", {"min": ov.min(), "mean": ov.mean(), "queries": int(ov.size),
                                              "below_0.99": int((ov < 0.99).sum())})
    assert ov.min() >= 0.99, (ov.min(), np.argsort(ov)[:5])


def test_c2_sparse(c2, decs):
    g, P = c2.g, c2.P
    dtype, dec, sdec = decs
    assert sdec.U_device.nnz == int(g["sparse_nnz"])
    idx, _ = topk_all(sdec, c2)
    ov = np.array([overlap(idx[j], g["top_sparse"][j]) for j in range(c2.batch.b)])
    record(f"{dtype}_sparse_end_to_end_top100_overlap", {"min": ov.min(), "mean": ov.mean(),
                                                         "below_0.99": int((ov < 0.99).sum())})
    nx = g["x_sparse"].shape[0]
    if dtype == "float64":
        Uh = sdec.U
        assert support_hash(Uh, P["r"]) == str(g["sparse_hash"])
        np.testing.assert_allclose(sdec.eta, g["sparse_eta"], rtol=1e-8, atol=1e-12)
        X = ranking.filter_batch(sdec, c2.h, first_queries(c2, nx))
        errs = [rel_l2(X[j], g["x_sparse"][j]) for j in range(nx)]
        record("float64_sparse_x_rel_l2_max", max(errs))
        assert max(errs) <= 1e-9, errs
        assert ov.min() >= 0.99, (ov.min(), np.argsort(ov)[:5])
        c2.support64 = Uh  # the reference's support (hash-pinned above)
    else:
        assert ov.mean() >= 0.99, ov.mean()


def test_c2_sparse_support_aligned_fp32(c2, decs):
    """fp32 values on the reference's kept (row, col) set: isolates kernel
    arithmetic from tau-boundary flips."""
    g = c2.g
    dtype, dec, _ = decs
    if dtype != "float32":
        pytest.skip("support-aligned check is for the fp32 pipeline")
    sup = getattr(c2, "support64", None)
    if sup is None:
        pytest.skip("fp64 support not available (fp64 case did not run)")
    U32 = dec.U  # host n x r fp32 values
    coo = sup.tocoo()
    Ua = sp.csr_matrix((U32[coo.row, coo.col].astype(np.float64), (coo.row, coo.col)), shape=sup.shape)
    Ua.sort_indices()
    eta = np.sqrt(np.asarray(Ua.multiply(Ua).sum(axis=1)).ravel())
    host = SimpleNamespace(U=Ua, eigenvalues=dec.eigenvalues, eta=eta, variant="sparse", provenance=None,
                           components=None)
    da = spectral.SpectralDecomposition.from_host(host, dtype="float32")
    nx = g["x_sparse"].shape[0]
    X = ranking.filter_batch(da, c2.h, first_queries(c2, nx))
    errs = [rel_l2(X[j], g["x_sparse"][j]) for j in range(nx)]
    record("float32_sparse_support_aligned_x_rel_l2_max", max(errs))
    assert max(errs) <= 1e-4, errs
    idx, _ = topk_all(da, c2)
    ov = np.array([overlap(idx[j], g["top_sparse"][j]) for j in range(c2.batch.b)])
    record("float32_sparse_support_aligned_top100_overlap", {"min": ov.min(), "mean": ov.mean()})
    assert ov.min() >= 0.99, (ov.min(), np.argsort(ov)[:5])
