"""Generate the golden fixtures under tests/golden from the REFERENCE itself.

Run in the build container only (it imports ``specrank`` from
/root/reference/pkg/src, which does not exist on the GPU box):

    python tests/golden/make_golden.py

The fixtures pin both the CPU oracle (tests/test_oracle.py) and the CUDA path
(tests/test_gpu_*.py).  Inputs are seeded (paper_1703_06935_b200.workloads).
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np
import scipy.sparse as sp

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

from specrank import graph, ranking, spectral  # noqa: E402
from specrank.descriptors import DescriptorSet  # noqa: E402
from specrank.sparsemat import SparseSymmetricMatrix  # noqa: E402

from paper_1703_06935_b200.workloads import CONFIGS, REGIONAL, cluster_descriptors, regional_descriptors  # noqa: E402


def support_hash(flat_sorted: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(flat_sorted, dtype=np.int64).tobytes()).hexdigest()


def csr_support(U) -> np.ndarray:
    coo = U.tocoo()
    return np.sort(coo.row.astype(np.int64) * U.shape[1] + coo.col.astype(np.int64))


def gaussian_cases():
    cases = [(7, 5, 0), (3, 3, 1), (64, 10, 12345), (33, 7, 2 ** 40 + 3), (1, 1, 7)]
    out = {}
    for i, (r, c, s) in enumerate(cases):
        out[f"g{i}_shape"] = np.array([r, c, s], dtype=np.uint64)
        out[f"g{i}"] = spectral.gaussian_matrix(r, c, s)
        gen = np.random.Generator(np.random.Philox(s))
        out[f"g{i}_uniforms"] = gen.random(16)
    out["count"] = np.array(len(cases))
    np.savez_compressed(os.path.join(HERE, "gaussian.npz"), **out)


def random_adjacency(n: int, density: float, seed: int):
    rng = np.random.default_rng(seed)
    M = rng.random((n, n)) * (rng.random((n, n)) < density)
    M = np.triu(M, 1)
    M = M + M.T
    return SparseSymmetricMatrix.from_dense(M)


def kat_cases():
    out = {}
    # rank-3 A = X X^T, r_hat=5, q=3 -> ||A - QQ^T A||_2 < 1e-8
    rng = np.random.default_rng(11)
    X = rng.standard_normal((64, 3))
    A = SparseSymmetricMatrix.from_dense(X @ X.T)
    basis = spectral.range_finder(A, 5, 3, 0)
    out["rank3_A"] = A.to_dense()
    out["rank3_Q"] = basis.Q
    out["rank3_B"] = basis.B

    # 2-node edge: Lambda = {1, -1}
    W2 = SparseSymmetricMatrix.from_dense(np.array([[0.0, 1.0], [1.0, 0.0]]))
    d2 = spectral.decompose(W2, 2, p=0, q=3, seed=0)
    out["two_U"] = d2.U
    out["two_lam"] = d2.eigenvalues

    # random normalized W, n=64, r=16
    Wr = random_adjacency(64, 0.15, 5)
    Sr = graph.normalize_adjacency(Wr, graph.degrees(Wr))
    dr = spectral.decompose(Sr, 16, p=10, q=4, seed=3)
    out["rand_W_dense"] = Sr.to_dense()
    out["rand_U"] = dr.U
    out["rand_lam"] = dr.eigenvalues
    out["rand_eta"] = dr.eta
    sp_dec = spectral.sparsify(dr, 200)
    out["rand_sparse_flat"] = csr_support(sp_dec.U)
    out["rand_sparse_eta"] = sp_dec.eta
    y = ranking.ObservationVector(64, np.array([1, 5, 9, 40]), np.array([0.5, 0.25, 1.0, 0.125]), cap=4)
    h = ranking.h_alpha(0.99)
    out["rand_y_idx"] = y.indices
    out["rand_y_val"] = y.values
    out["rand_x_approx"] = ranking.filter(dr, h, y)
    out["rand_x_sparse"] = ranking.filter(sp_dec, h, y)
    heat = ranking.custom_transfer(lambda x: np.exp(-10.0 * (1.0 - x)), nondecreasing=True, positive=True)
    out["rand_x_heat"] = ranking.filter(dr, heat, y)

    # n=12 graph with an isolated vertex -> eta = 0 rows exercise copy_uncovered
    Wi = random_adjacency(12, 0.5, 9).to_dense()
    Wi[3, :] = 0.0
    Wi[:, 3] = 0.0
    Wi = SparseSymmetricMatrix.from_dense(Wi)
    Si = graph.normalize_adjacency(Wi, graph.degrees(Wi))
    di = spectral.decompose(Si, 6, p=2, q=3, seed=1)
    yi = ranking.ObservationVector(12, np.array([0, 3, 7]), np.array([1.0, 2.0, 0.5]), cap=3)
    out["iso_W_dense"] = Si.to_dense()
    out["iso_lam"] = di.eigenvalues
    out["iso_eta"] = di.eta
    out["iso_x"] = ranking.filter(di, h, yi)
    si = spectral.sparsify(di, 30)  # row 3 keeps nothing -> eta == 0 exactly
    out["iso_sparse_eta"] = si.eta
    out["iso_sparse_flat"] = csr_support(si.U)
    out["iso_x_sparse"] = ranking.filter(si, h, yi)
    out["iso_y_idx"] = yi.indices
    out["iso_y_val"] = yi.values
    np.savez_compressed(os.path.join(HERE, "kat.npz"), **out)


def c1_case(n_x: int = 20):
    cfg = CONFIGS["C1"]
    t0 = time.perf_counter()
    data, queries, _ = cluster_descriptors(cfg)
    ds = DescriptorSet(data)
    W = graph.build_mutual_knn_graph(ds, cfg.k, cfg.gamma)
    S = graph.normalize_adjacency(W, graph.degrees(W))
    t1 = time.perf_counter()
    dec = spectral.decompose(S, cfg.r, p=cfg.p, q=cfg.q, seed=0)
    t2 = time.perf_counter()
    sdec = spectral.sparsify(dec, cfg.tau)
    t3 = time.perf_counter()
    h = ranking.h_alpha(cfg.alpha)
    ys = [ranking.observation_vector(qv, ds, cfg.y_top, cfg.gamma) for qv in queries]
    y_ptr = np.zeros(len(ys) + 1, dtype=np.int64)
    y_ptr[1:] = np.cumsum([y.nnz for y in ys])
    y_idx = np.concatenate([y.indices for y in ys])
    y_val = np.concatenate([y.values for y in ys])
    top_a, top_s, xa, xs = [], [], [], []
    for j, y in enumerate(ys):
        x = ranking.filter(dec, h, y)
        x2 = ranking.filter(sdec, h, y)
        top_a.append(ranking.rank(x)[:100])
        top_s.append(ranking.rank(x2)[:100])
        if j < n_x:
            xa.append(x)
            xs.append(x2)
    t4 = time.perf_counter()
    flat = csr_support(sdec.U)
    print(f"C1: graph {t1 - t0:.1f}s decompose {t2 - t1:.1f}s sparsify {t3 - t2:.1f}s "
          f"queries {t4 - t3:.1f}s nnz(W)={W.nnz}")
    np.savez_compressed(
        os.path.join(HERE, "c1.npz"),
        W_indptr=W.csr.indptr.astype(np.int64), W_indices=W.csr.indices.astype(np.int32),
        W_data=W.csr.data, S_data=S.csr.data,
        lam=dec.eigenvalues, eta=dec.eta, U_cols=dec.U[:, :4].copy(),
        U_colsum_abs=np.abs(dec.U).sum(axis=0),
        sparse_eta=sdec.eta, sparse_nnz=np.array(sdec.U.nnz),
        sparse_hash=np.array(support_hash(flat)),
        sparse_flat_head=flat[:2000],
        y_ptr=y_ptr, y_idx=y_idx, y_val=y_val,
        x_approx=np.array(xa), x_sparse=np.array(xs),
        top_approx=np.array(top_a, dtype=np.int32), top_sparse=np.array(top_s, dtype=np.int32),
        params=np.array([cfg.n, cfg.r, cfg.p, cfg.q, cfg.tau, 0]),
        alpha=np.array(cfg.alpha),
    )


def epilogue_case(n_q: int = 5, region_per_image: int = 4):
    """FSRw, pooling and the embedding on the C1 decomposition."""
    cfg = CONFIGS["C1"]
    data, queries, _ = cluster_descriptors(cfg)
    ds = DescriptorSet(data)
    W = graph.build_mutual_knn_graph(ds, cfg.k, cfg.gamma)
    S = graph.normalize_adjacency(W, graph.degrees(W))
    dec = spectral.decompose(S, cfg.r, p=cfg.p, q=cfg.q, seed=0)
    sdec = spectral.sparsify(dec, cfg.tau)
    h = ranking.h_alpha(cfg.alpha)
    n = cfg.n
    rng = np.random.default_rng(11)
    r2i = np.arange(n) // region_per_image
    wts = rng.uniform(0.5, 1.5, n)
    P = ranking.PoolingMatrix.from_region_map(r2i, weights=wts)
    out = {"r2i": r2i, "pool_w": wts}
    for tag, d in (("a", dec), ("s", sdec)):
        xs, xw, xp, xf, order = [], [], [], [], []
        Ub = ranking.pooled_basis(P, d)
        for j in range(n_q):
            y = ranking.observation_vector(queries[j], ds, cfg.y_top, cfg.gamma)
            x = ranking.filter(d, h, y)
            xs.append(x)
            xw.append(ranking.fsrw_correct(x, d, ds, queries[j]))
            xp.append(ranking.pool(P, x))
            xf.append(ranking.filter_pooled(d, h, y, Ub))
            order.append(ranking.RankingResult.from_scores(x, P).order[:100])
        out[f"{tag}_fsrw"] = np.array(xw)
        out[f"{tag}_pool"] = np.array(xp)
        out[f"{tag}_filter_pooled"] = np.array(xf)
        out[f"{tag}_pooled_order"] = np.array(order)
        out[f"{tag}_ubar_head"] = Ub[:200].copy()
        out[f"{tag}_ubar_rowsum"] = Ub.sum(axis=1)
        out[f"{tag}_ubar_colsum"] = Ub.sum(axis=0)
        phi = ranking.embedding(d, h)
        sims = [ranking.out_of_sample_similarity(queries[a], queries[b], phi, ds, cfg.y_top, cfg.gamma)
                for a, b in ((0, 1), (2, 3), (4, 4), (5, 9))]
        out[f"{tag}_oos"] = np.array(sims)
    np.savez_compressed(os.path.join(HERE, "epi.npz"), **out)


def c2_reduced_case(n: int = 20_000, queries: int = 50, r: int = 400, p: int = 40, n_x: int = 5):
    """C2's generator (d=512, 1000 Zipf clusters, k=50, gamma=3, tau=5%) at n=20k
    (reduced C2), r=400, p=40, q=3."""
    from dataclasses import replace

    cfg = replace(CONFIGS["C2"], n=n, queries=queries, r=r, p=p)
    t0 = time.perf_counter()
    data, qv, _ = cluster_descriptors(cfg)
    ds = DescriptorSet(data)
    W = graph.build_mutual_knn_graph(ds, cfg.k, cfg.gamma)
    S = graph.normalize_adjacency(W, graph.degrees(W))
    t1 = time.perf_counter()
    dec = spectral.decompose(S, cfg.r, p=cfg.p, q=cfg.q, seed=0)
    sdec = spectral.sparsify(dec, cfg.tau)
    h = ranking.h_alpha(cfg.alpha)
    ys = [ranking.observation_vector(q, ds, cfg.y_top, cfg.gamma) for q in qv]
    y_ptr = np.zeros(len(ys) + 1, dtype=np.int64)
    y_ptr[1:] = np.cumsum([y.nnz for y in ys])
    xa, xs, ta, ts = [], [], [], []
    for j, y in enumerate(ys):
        x = ranking.filter(dec, h, y)
        x2 = ranking.filter(sdec, h, y)
        ta.append(ranking.rank(x)[:100])
        ts.append(ranking.rank(x2)[:100])
        if j < n_x:
            xa.append(x)
            xs.append(x2)
    flat = csr_support(sdec.U)
    print(f"C2r: graph {t1 - t0:.1f}s total {time.perf_counter() - t0:.1f}s nnz(W)={W.nnz}")
    np.savez_compressed(
        os.path.join(HERE, "c2r.npz"),
        W_indptr=W.csr.indptr.astype(np.int64), W_indices=W.csr.indices.astype(np.int32),
        S_data=S.csr.data, lam=dec.eigenvalues, eta=dec.eta, sparse_eta=sdec.eta,
        sparse_nnz=np.array(sdec.U.nnz), sparse_hash=np.array(support_hash(flat)),
        y_ptr=y_ptr, y_idx=np.concatenate([y.indices for y in ys]), y_val=np.concatenate([y.values for y in ys]),
        x_approx=np.array(xa), x_sparse=np.array(xs),
        top_approx=np.array(ta, dtype=np.int32), top_sparse=np.array(ts, dtype=np.int32),
        params=np.array([cfg.n, cfg.r, cfg.p, cfg.q, cfg.tau, 0]), alpha=np.array(cfg.alpha),
    )


def weight_digest(data: np.ndarray) -> np.ndarray:
    """Size-independent digest of a CSR value array in its stored order:
    [sum, sum of squares, sum weighted by seeded U(0,1) coefficients, max].
    Two arrays whose entries agree to 1e-12 relative agree to ~1e-12 here;
    a single wrong entry moves the weighted sum."""
    c = np.random.default_rng(99).random(data.size)
    return np.array([data.sum(), np.dot(data, data), np.dot(data, c), data.max() if data.size else 0.0])


def pattern_hash(indptr: np.ndarray, indices: np.ndarray) -> str:
    h = hashlib.sha256(np.ascontiguousarray(indptr, dtype=np.int64).tobytes())
    h.update(np.ascontiguousarray(indices, dtype=np.int32).tobytes())
    return h.hexdigest()


def c2_full_case(n_x: int = 4, top: int = 100):
    """BASELINE C2 at full size (n=1e5, d=512, 1000 Zipf clusters, k=50,
    gamma=3, r=2000, p=200, q=3, tau=5% = 1e7, 1000 queries, y top-50,
    h_alpha(0.99)), run through the reference.  Only outputs are stored (no
    W: 2.7e6 fp64 weights); the GPU test regenerates W from the seeded
    descriptors with the fp64 device builder and checks it against
    ``W_pattern_hash`` / ``W_digest``.  Also records the reference's own
    stage timings in this container (8 cores, OpenBLAS)."""
    cfg = CONFIGS["C2"]
    tm = {}
    t0 = time.perf_counter()
    data, qv, _ = cluster_descriptors(cfg)
    ds = DescriptorSet(data)
    W = graph.build_mutual_knn_graph(ds, cfg.k, cfg.gamma)
    S = graph.normalize_adjacency(W, graph.degrees(W))
    tm["graph"] = time.perf_counter() - t0
    t = time.perf_counter()
    basis = spectral.range_finder(S, cfg.r_hat, cfg.q, 0)
    tm["range_finder"] = time.perf_counter() - t
    t = time.perf_counter()
    dec = spectral.approx_eigendecomposition(S, basis, cfg.r)
    tm["approx_eig"] = time.perf_counter() - t
    del basis
    t = time.perf_counter()
    sdec = spectral.sparsify(dec, cfg.tau)
    tm["sparsify"] = time.perf_counter() - t
    h = ranking.h_alpha(cfg.alpha)
    t = time.perf_counter()
    ys = [ranking.observation_vector(q, ds, cfg.y_top, cfg.gamma) for q in qv]
    tm["observation_vectors"] = time.perf_counter() - t
    y_ptr = np.zeros(len(ys) + 1, dtype=np.int64)
    y_ptr[1:] = np.cumsum([y.nnz for y in ys])
    xa, xs, ta, ts, va, vs = [], [], [], [], [], []
    tf = [0.0, 0.0]
    for j, y in enumerate(ys):
        t = time.perf_counter()
        x = ranking.filter(dec, h, y)
        tf[0] += time.perf_counter() - t
        t = time.perf_counter()
        x2 = ranking.filter(sdec, h, y)
        tf[1] += time.perf_counter() - t
        oa, os_ = ranking.rank(x)[:top + 1], ranking.rank(x2)[:top + 1]
        ta.append(oa[:top])
        ts.append(os_[:top])
        va.append(x[oa])
        vs.append(x2[os_])
        if j < n_x:
            xa.append(x)
            xs.append(x2)
    tm["filter_dense_per_query"] = tf[0] / len(ys)
    tm["filter_sparse_per_query"] = tf[1] / len(ys)
    flat = csr_support(sdec.U)
    print(f"C2: {tm} nnz(W)={W.nnz}")
    np.savez_compressed(
        os.path.join(HERE, "c2.npz"),
        W_nnz=np.array(W.nnz), W_pattern_hash=np.array(pattern_hash(W.csr.indptr, W.csr.indices)),
        W_digest=weight_digest(W.csr.data), S_digest=weight_digest(S.csr.data),
        lam=dec.eigenvalues, eta=dec.eta, sparse_eta=sdec.eta,
        U_colsum_abs=np.abs(dec.U).sum(axis=0),
        sparse_nnz=np.array(sdec.U.nnz), sparse_hash=np.array(support_hash(flat)),
        y_ptr=y_ptr, y_idx=np.concatenate([y.indices for y in ys]), y_val=np.concatenate([y.values for y in ys]),
        x_approx=np.array(xa), x_sparse=np.array(xs),
        top_approx=np.array(ta, dtype=np.int32), top_sparse=np.array(ts, dtype=np.int32),
        topval_approx=np.array(va), topval_sparse=np.array(vs),
        params=np.array([cfg.n, cfg.r, cfg.p, cfg.q, cfg.tau, 0]), alpha=np.array(cfg.alpha),
        timings_keys=np.array(list(tm.keys())), timings=np.array(list(tm.values())),
        host=np.array(f"{os.cpu_count()} cores, numpy {np.__version__}"),
    )


def c4_reduced_case(n_x: int = 5):
    """C4's regional generator (images x 5 regions, sigma=0.05, d=512, k=50,
    gamma=3, tau=2%) at 4000 images (n = 20k), r=400, p=40, q=3; queries pool
    their 5 regions into one observation vector (cap 50); region scores are
    also pooled to images (PoolingMatrix, RankingResult)."""
    cfg = REGIONAL["C4r"]
    t0 = time.perf_counter()
    data, qx, r2i, qimg = regional_descriptors(cfg)
    ds = DescriptorSet(data)
    W = graph.build_mutual_knn_graph(ds, cfg.k, cfg.gamma)
    S = graph.normalize_adjacency(W, graph.degrees(W))
    t1 = time.perf_counter()
    dec = spectral.decompose(S, cfg.r, p=cfg.p, q=cfg.q, seed=0)
    sdec = spectral.sparsify(dec, cfg.tau)
    h = ranking.h_alpha(cfg.alpha)
    m = cfg.regions
    ys = [ranking.observation_vector(qx[j * m:(j + 1) * m], ds, cfg.y_top, cfg.gamma, cap=cfg.y_top)
          for j in range(cfg.queries)]
    y_ptr = np.zeros(len(ys) + 1, dtype=np.int64)
    y_ptr[1:] = np.cumsum([y.nnz for y in ys])
    P = ranking.PoolingMatrix.from_region_map(r2i)
    xa, xs, ta, ts, ia, isp = [], [], [], [], [], []
    for j, y in enumerate(ys):
        x = ranking.filter(dec, h, y)
        x2 = ranking.filter(sdec, h, y)
        ta.append(ranking.rank(x)[:100])
        ts.append(ranking.rank(x2)[:100])
        ia.append(ranking.RankingResult.from_scores(x, P).order[:100])
        isp.append(ranking.RankingResult.from_scores(x2, P).order[:100])
        if j < n_x:
            xa.append(x)
            xs.append(x2)
    flat = csr_support(sdec.U)
    print(f"C4r: graph {t1 - t0:.1f}s total {time.perf_counter() - t0:.1f}s nnz(W)={W.nnz}")
    np.savez_compressed(
        os.path.join(HERE, "c4r.npz"),
        W_indptr=W.csr.indptr.astype(np.int64), W_indices=W.csr.indices.astype(np.int32),
        W_data=W.csr.data, lam=dec.eigenvalues, eta=dec.eta, sparse_eta=sdec.eta,
        sparse_nnz=np.array(sdec.U.nnz), sparse_hash=np.array(support_hash(flat)),
        y_ptr=y_ptr, y_idx=np.concatenate([y.indices for y in ys]), y_val=np.concatenate([y.values for y in ys]),
        x_approx=np.array(xa), x_sparse=np.array(xs),
        top_approx=np.array(ta, dtype=np.int32), top_sparse=np.array(ts, dtype=np.int32),
        img_top_approx=np.array(ia, dtype=np.int32), img_top_sparse=np.array(isp, dtype=np.int32),
        query_images=qimg, params=np.array([cfg.n, cfg.r, cfg.p, cfg.q, cfg.tau, 0]), alpha=np.array(cfg.alpha),
    )


def block_graph(sizes, seed: int, density: float = 0.08):
    """Symmetric nonnegative adjacency whose components have the given sizes
    (each block connected: a random spanning path plus random edges), vertices
    randomly permuted so the labeling is not trivial."""
    rng = np.random.default_rng(seed)
    n = int(sum(sizes))
    perm = rng.permutation(n)
    rows, cols = [], []
    start = 0
    for m in sizes:
        v = perm[start:start + m]
        start += m
        if m == 1:
            continue
        for a in range(m - 1):  # spanning path keeps the block connected
            rows.append(v[a]), cols.append(v[a + 1])
        extra = rng.random((m, m)) < density
        ii, jj = np.nonzero(np.triu(extra, 1))
        rows.extend(v[ii].tolist()), cols.extend(v[jj].tolist())
    rows, cols = np.array(rows, dtype=np.int64), np.array(cols, dtype=np.int64)
    vals = rng.uniform(0.1, 1.0, rows.size)
    W = sp.coo_matrix((np.r_[vals, vals], (np.r_[rows, cols], np.r_[cols, rows])), shape=(n, n)).tocsr()
    W.sum_duplicates()
    W.sort_indices()
    return W


def blockwise_case():
    """connected_components + decompose_blockwise + exact/rank-r decompositions."""
    W = block_graph([300, 120, 45, 30, 2, 2, 1, 1, 1], seed=21)
    A = SparseSymmetricMatrix(W)
    lab = graph.connected_components(A)
    S = graph.normalize_adjacency(A, graph.degrees(A))
    out = {"W_indptr": W.indptr.astype(np.int64), "W_indices": W.indices.astype(np.int32), "W_data": W.data,
           "S_data": S.csr.data, "labels": lab.labels, "sizes": lab.sizes, "order": lab.order}
    for tag, rho, r in (("mixed", 50, 60), ("exact", 400, 60)):
        # step r down until the r-th and (r+1)-th candidates are well separated
        while True:
            dec = spectral.decompose_blockwise(S, lab, r=r, rho=rho, p=10, q=4, seed=7)
            full = spectral.decompose_blockwise(S, lab, r=10 ** 6, rho=rho, p=10, q=4, seed=7)
            lam_all = full.eigenvalues
            if r >= lam_all.size or lam_all[r - 1] - lam_all[r] > 1e-6:
                break
            r -= 1
        out[f"{tag}_r"] = np.array(r)
        out[f"{tag}_lam"] = dec.eigenvalues
        out[f"{tag}_U"] = dec.dense_u()
        out[f"{tag}_eta"] = dec.eta
        out[f"{tag}_variant"] = np.array(dec.variant.value)
    sub = A.submatrix(lab.vertices_of(2))
    ex = spectral.exact_eigendecomposition(graph.normalize_adjacency(sub, graph.degrees(sub)))
    out["exact_sub_lam"], out["exact_sub_U"] = ex.eigenvalues, ex.U
    rr = spectral.rank_r_decomposition(S.submatrix(lab.vertices_of(1)), 17)
    out["rankr_lam"], out["rankr_U"], out["rankr_eta"] = rr.eigenvalues, rr.U, rr.eta
    np.savez_compressed(os.path.join(HERE, "blockwise.npz"), **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["gaussian", "kat", "c1", "epi", "blockwise", "c2r", "c4r"]
    if "gaussian" in which:
        gaussian_cases()
    if "kat" in which:
        kat_cases()
    if "c1" in which:
        c1_case()
    if "epi" in which:
        epilogue_case()
    if "blockwise" in which:
        blockwise_case()
    if "c2r" in which:
        c2_reduced_case()
    if "c4r" in which:
        c4_reduced_case()
    if "c2" in which:  # full BASELINE C2: ~25 min on 8 cores, run explicitly
        c2_full_case()
    print("ok")
