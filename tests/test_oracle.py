"""Pin the CPU oracle against fixtures produced by the reference itself."""

import numpy as np
import scipy.sparse as sp

from oracle import fsr_oracle as O


def c1_matrices(g):
    n = int(g["params"][0])
    W = sp.csr_matrix((g["W_data"], g["W_indices"], g["W_indptr"]), shape=(n, n))
    S = sp.csr_matrix((g["S_data"], g["W_indices"], g["W_indptr"]), shape=(n, n))
    return W, S


def test_philox_block_matches_numpy_stream():
    for seed in (0, 1, 12345, 2 ** 40 + 3):
        raw = np.random.Philox(seed).random_raw(8)
        key = O.philox_key(seed)
        mine = [O.philox4x64_10((1, 0, 0, 0), key), O.philox4x64_10((2, 0, 0, 0), key)]
        assert [int(v) for v in raw] == [int(v) for blk in mine for v in blk]


def test_gaussian_matches_reference(golden):
    g = golden("gaussian")
    for i in range(int(g["count"])):
        r, c, s = (int(v) for v in g[f"g{i}_shape"])
        np.testing.assert_array_equal(O.gaussian_matrix(r, c, s), g[f"g{i}"])
        np.testing.assert_array_equal(O.philox_uniforms(s, 0, 16), g[f"g{i}_uniforms"])


def test_normalize_matches_reference_bitwise(golden):
    g = golden("c1")
    W, S = c1_matrices(g)
    S2 = O.normalize_adjacency(W, O.degrees(W))
    S2.sort_indices()
    np.testing.assert_array_equal(S2.indptr, S.indptr)
    np.testing.assert_array_equal(S2.data, S.data)


def test_kat_rank3_range_finder(golden):
    k = golden("kat")
    A = sp.csr_matrix(k["rank3_A"])
    Q, B = O.range_finder(A, 5, 3, 0)
    np.testing.assert_allclose(np.abs(Q.T @ k["rank3_Q"]).max(), 1.0, atol=1e-12)
    resid = np.linalg.norm(k["rank3_A"] - Q @ (Q.T @ k["rank3_A"]), 2)
    assert resid < 1e-8


def test_kat_two_node(golden):
    k = golden("kat")
    U, lam, eta = O.decompose(sp.csr_matrix(np.array([[0.0, 1.0], [1.0, 0.0]])), 2, p=0, q=3, seed=0)
    np.testing.assert_allclose(lam, [1.0, -1.0], atol=1e-12)
    np.testing.assert_allclose(lam, k["two_lam"], atol=1e-14)
    np.testing.assert_allclose(U, k["two_U"], atol=1e-12)


def test_kat_random_and_filter(golden):
    k = golden("kat")
    S = sp.csr_matrix(k["rand_W_dense"])
    U, lam, eta = O.decompose(S, 16, p=10, q=4, seed=3)
    np.testing.assert_allclose(lam, k["rand_lam"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(U, k["rand_U"], atol=1e-10)
    Ut, eta_s = O.sparsify(U, 200)
    coo = Ut.tocoo()
    np.testing.assert_array_equal(np.sort(coo.row.astype(np.int64) * 16 + coo.col), k["rand_sparse_flat"])
    np.testing.assert_array_equal(O.sparsify_support(U, 200), k["rand_sparse_flat"])
    w = O.transfer_values(O.h_alpha(0.99), lam)
    x = O.filter_scores(U, lam, eta, w, k["rand_y_idx"], k["rand_y_val"])
    np.testing.assert_allclose(x, k["rand_x_approx"], rtol=1e-10, atol=1e-13)
    xs = O.filter_scores(Ut, lam, eta_s, w, k["rand_y_idx"], k["rand_y_val"])
    np.testing.assert_allclose(xs, k["rand_x_sparse"], rtol=1e-10, atol=1e-13)
    wh = O.transfer_values(O.heat_kernel(10.0), lam, analytic=False)
    xh = O.filter_scores(U, lam, eta, wh, k["rand_y_idx"], k["rand_y_val"])
    np.testing.assert_allclose(xh, k["rand_x_heat"], rtol=1e-10, atol=1e-13)


def test_kat_isolated_vertex_copy_uncovered(golden):
    k = golden("kat")
    U, lam, eta = O.decompose(sp.csr_matrix(k["iso_W_dense"]), 6, p=2, q=3, seed=1)
    w = O.transfer_values(O.h_alpha(0.99), lam)
    x = O.filter_scores(U, lam, eta, w, k["iso_y_idx"], k["iso_y_val"])
    np.testing.assert_allclose(x, k["iso_x"], rtol=1e-10, atol=1e-13)
    Ut, eta_s = O.sparsify(U, 30)
    assert eta_s[3] == 0.0
    np.testing.assert_array_equal(eta_s, k["iso_sparse_eta"])
    xs = O.filter_scores(Ut, lam, eta_s, w, k["iso_y_idx"], k["iso_y_val"])
    np.testing.assert_allclose(xs, k["iso_x_sparse"], rtol=1e-10, atol=1e-13)
    assert xs[3] == 2.0


def test_c1_oracle_matches_reference(golden):
    g = golden("c1")
    _, S = c1_matrices(g)
    n, r, p, q, tau, seed = (int(v) for v in g["params"])
    U, lam, eta = O.decompose(S, r, p=p, q=q, seed=seed)
    np.testing.assert_allclose(lam, g["lam"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(eta, g["eta"], atol=1e-10)
    w = O.transfer_values(O.h_alpha(float(g["alpha"])), lam)
    for j in range(3):
        sl = slice(g["y_ptr"][j], g["y_ptr"][j + 1])
        x = O.filter_scores(U, lam, eta, w, g["y_idx"][sl], g["y_val"][sl])
        np.testing.assert_allclose(x, g["x_approx"][j], rtol=1e-8, atol=1e-12)
    flat = O.sparsify_support(U, tau)
    assert flat.size == int(g["sparse_nnz"])
    import hashlib
    assert hashlib.sha256(flat.astype(np.int64).tobytes()).hexdigest() == str(g["sparse_hash"])


def test_c1_oracle_epilogues_match_reference(golden):
    """FSRw, pooling, filter_pooled and the embedding similarity (ranking.py:256-387)
    restated by the oracle on its own C1 decomposition vs the reference's outputs."""
    import os
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_1703_06935_b200.workloads import CONFIGS, cluster_descriptors

    g, e = golden("c1"), golden("epi")
    cfg = CONFIGS["C1"]
    data, queries, _ = cluster_descriptors(cfg)
    _, S = c1_matrices(g)
    n, r, p, q, tau, seed = (int(v) for v in g["params"])
    U, lam, eta = O.decompose(S, r, p=p, q=q, seed=seed)
    Us, eta_s = O.sparsify(U, tau)
    w = O.transfer_values(O.h_alpha(float(g["alpha"])), lam)
    P = O.pooling_from_region_map(e["r2i"], weights=e["pool_w"])
    for tag, UU, et in (("a", U, eta), ("s", Us, eta_s)):
        Ub = O.pooled_basis(P, UU)
        np.testing.assert_allclose(Ub[:200], e[f"{tag}_ubar_head"], rtol=1e-8, atol=1e-12)
        np.testing.assert_allclose(Ub.sum(axis=1), e[f"{tag}_ubar_rowsum"], rtol=1e-8, atol=1e-11)
        for j in range(e[f"{tag}_fsrw"].shape[0]):
            yi, yv = O.observation_vector(queries[j], data, cfg.y_top, cfg.gamma)
            x = O.filter_scores(UU, lam, et, w, yi, yv)
            np.testing.assert_allclose(O.fsrw_correct(x, et, data, queries[j]), e[f"{tag}_fsrw"][j],
                                       rtol=1e-8, atol=1e-12)
            xp = O.pool(P, x)
            np.testing.assert_allclose(xp, e[f"{tag}_pool"][j], rtol=1e-8, atol=1e-12)
            np.testing.assert_array_equal(O.rank(xp)[:100], e[f"{tag}_pooled_order"][j])
            np.testing.assert_allclose(O.filter_pooled(UU, w, yi, yv, Ub), e[f"{tag}_filter_pooled"][j],
                                       rtol=1e-8, atol=1e-12)
        phi = O.embedding(UU, w)
        sims = [O.out_of_sample_similarity(queries[a], queries[b], phi, data, cfg.y_top, cfg.gamma)
                for a, b in ((0, 1), (2, 3), (4, 4), (5, 9))]
        np.testing.assert_allclose(sims, e[f"{tag}_oos"], rtol=1e-8)


def _blockwise_mats(b):
    n = b["labels"].size
    W = sp.csr_matrix((b["W_data"], b["W_indices"], b["W_indptr"]), shape=(n, n))
    S = sp.csr_matrix((b["S_data"], b["W_indices"], b["W_indptr"]), shape=(n, n))
    return W, S


def _assert_same_spectral_operator(U, lam, U_ref, lam_ref, tol):
    """Invariant to column order among equal eigenvalues and to signs."""
    np.testing.assert_allclose(np.sort(lam)[::-1], np.sort(lam_ref)[::-1], atol=tol)
    np.testing.assert_allclose((U * lam) @ U.T, (U_ref * lam_ref) @ U_ref.T, atol=tol)
    np.testing.assert_allclose(U @ U.T, U_ref @ U_ref.T, atol=tol)


def test_oracle_components_and_blockwise_match_reference(golden):
    b = golden("blockwise")
    W, S = _blockwise_mats(b)
    labels, sizes, order = O.connected_components(W)
    np.testing.assert_array_equal(labels, b["labels"])
    np.testing.assert_array_equal(sizes, b["sizes"])
    np.testing.assert_array_equal(order, b["order"])
    for tag, rho in (("mixed", 50), ("exact", 400)):
        U, lam, eta, all_exact, truncated = O.decompose_blockwise(S, labels, int(b[f"{tag}_r"]), rho, p=10, q=4,
                                                                  seed=7)
        variant = ("rank_r" if truncated else "exact") if all_exact else "approx"
        assert variant == str(b[f"{tag}_variant"])
        _assert_same_spectral_operator(U, lam, b[f"{tag}_U"], b[f"{tag}_lam"], 1e-9)
        np.testing.assert_allclose(eta, b[f"{tag}_eta"], atol=1e-9)


def test_c2_reduced_oracle_matches_reference(golden):
    g = golden("c2r")
    n, r, p, q, tau, seed = (int(v) for v in g["params"])
    S = sp.csr_matrix((g["S_data"], g["W_indices"], g["W_indptr"]), shape=(n, n))
    U, lam, eta = O.decompose(S, r, p=p, q=q, seed=seed)
    np.testing.assert_allclose(lam, g["lam"], rtol=0, atol=1e-12)
    w = O.transfer_values(O.h_alpha(float(g["alpha"])), lam)
    sl = slice(g["y_ptr"][0], g["y_ptr"][1])
    x = O.filter_scores(U, lam, eta, w, g["y_idx"][sl], g["y_val"][sl])
    np.testing.assert_allclose(x, g["x_approx"][0], rtol=1e-8, atol=1e-12)
    import hashlib
    flat = O.sparsify_support(U, tau)
    assert hashlib.sha256(flat.astype(np.int64).tobytes()).hexdigest() == str(g["sparse_hash"])


def test_c4_reduced_oracle_matches_reference(golden):
    """Regional C4r: pooled 5-region observation vectors, normalisation,
    decomposition, sparse support and image pooling of the oracle against
    the reference's outputs (tests/golden/c4r.npz)."""
    import hashlib

    from paper_1703_06935_b200.workloads import REGIONAL, regional_descriptors

    g = golden("c4r")
    cfg = REGIONAL["C4r"]
    data, qx, r2i, qimg = regional_descriptors(cfg)
    np.testing.assert_array_equal(qimg, g["query_images"])
    m = cfg.regions
    for j in (0, 7, cfg.queries - 1):
        oi, ov = O.observation_vector(qx[j * m:(j + 1) * m], data, cfg.y_top, cfg.gamma, cap=cfg.y_top)
        sl = slice(g["y_ptr"][j], g["y_ptr"][j + 1])
        np.testing.assert_array_equal(oi, g["y_idx"][sl])
        np.testing.assert_allclose(ov, g["y_val"][sl], rtol=1e-13, atol=0)
    n = cfg.n
    W = sp.csr_matrix((g["W_data"], g["W_indices"], g["W_indptr"]), shape=(n, n))
    S = O.normalize_adjacency(W, O.degrees(W))
    U, lam, eta = O.decompose(S, cfg.r, p=cfg.p, q=cfg.q, seed=0)
    np.testing.assert_allclose(lam, g["lam"], rtol=0, atol=1e-12)
    flat = O.sparsify_support(U, cfg.tau)
    assert hashlib.sha256(flat.astype(np.int64).tobytes()).hexdigest() == str(g["sparse_hash"])
    w = O.transfer_values(O.h_alpha(float(g["alpha"])), lam)
    P = O.pooling_from_region_map(r2i)
    sl = slice(g["y_ptr"][0], g["y_ptr"][1])
    x = O.filter_scores(U, lam, eta, w, g["y_idx"][sl], g["y_val"][sl])
    np.testing.assert_allclose(x, g["x_approx"][0], rtol=1e-8, atol=1e-12)
    np.testing.assert_array_equal(O.rank(O.pool(P, x))[:100], g["img_top_approx"][0])
