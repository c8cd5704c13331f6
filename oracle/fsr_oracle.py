"""CPU oracle for the FSR hot path -- TEST INFRASTRUCTURE ONLY.

This module restates, in plain numpy/scipy, the reference algorithm of the
path the CUDA library accelerates.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it, and only as the checker or the
timed CPU baseline -- never as the product path.  The product
(``paper_1703_06935_b200``) never imports this package.

Pinning: the reference is pure Python (``/root/reference/pkg/src/specrank``)
and importable in the build container, so ``tests/golden/make_golden.py``
runs the reference itself on seeded inputs and commits the outputs under
``tests/golden``; ``tests/test_oracle.py`` checks this restatement against
those fixtures.  The reference's arithmetic lives in numpy 2.3.5 / scipy
1.18.1 (OpenBLAS LAPACK for QR/eigh, scipy sparsetools for CSR products), the
same libraries used here.

Every function cites the reference file:line it restates (paths relative to
``/root/reference/pkg/src/specrank``).
"""

from __future__ import annotations

import warnings

import numpy as np
import scipy.sparse as sp

MASK64 = (1 << 64) - 1

# ---------------------------------------------------------------------------
# Philox4x64-10 (numpy's counter-based generator, used by gaussian_matrix)
# ---------------------------------------------------------------------------
PHILOX_M0 = 0xD2E7470EE14C6C93
PHILOX_M1 = 0xCA5A826395121157
PHILOX_W0 = 0x9E3779B97F4A7C15
PHILOX_W1 = 0xBB67AE8584CAA73B


def philox4x64_10(counter, key):
    """One Philox4x64 block with 10 rounds (Salmon et al., SC'11; numpy's
    ``Philox`` bit generator).  ``counter`` is 4 ints, ``key`` 2 ints."""
    c0, c1, c2, c3 = (int(v) & MASK64 for v in counter)
    k0, k1 = (int(v) & MASK64 for v in key)
    for rnd in range(10):
        if rnd:
            k0 = (k0 + PHILOX_W0) & MASK64
            k1 = (k1 + PHILOX_W1) & MASK64
        p0 = PHILOX_M0 * c0
        p1 = PHILOX_M1 * c2
        c0, c1, c2, c3 = ((p1 >> 64) ^ c1 ^ k0, p1 & MASK64,
                          (p0 >> 64) ^ c3 ^ k1, p0 & MASK64)
    return c0, c1, c2, c3


def philox_key(seed: int):
    """Key numpy derives for ``Philox(seed)``: SeedSequence(seed) state words."""
    return tuple(int(v) for v in np.random.SeedSequence(seed & MASK64).generate_state(2, np.uint64))


def philox_uniforms(seed: int, start: int, count: int) -> np.ndarray:
    """Uniform doubles ``start .. start+count-1`` of ``Generator(Philox(seed)).random``.

    The generator emits one Philox block per counter value, the first block
    at counter 1, and ``random()`` maps a draw x to ``(x >> 11) * 2**-53``.
    Pure-Python (slow): for small pins only.
    """
    key = philox_key(seed)
    out = np.empty(count)
    for i in range(count):
        m = start + i
        blk = philox4x64_10((m // 4 + 1, 0, 0, 0), key)
        out[i] = (blk[m % 4] >> 11) * (2.0 ** -53)
    return out


def gaussian_matrix(rows: int, cols: int, seed: int) -> np.ndarray:
    """Box-Muller Gaussian block (``spectral.py:55-65``).

    ``half = ceil(count/2)`` uniforms feed the radii (as ``1 - u``) and the
    next ``half`` feed the angles; the output is ``concat(r cos, r sin)``
    truncated to ``count`` and laid out row-major.
    """
    gen = np.random.Generator(np.random.Philox(seed & MASK64))
    count = rows * cols
    half = (count + 1) // 2
    u_radius = 1.0 - gen.random(half)
    u_angle = gen.random(half)
    rad = np.sqrt(-2.0 * np.log(u_radius))
    ang = 2.0 * np.pi * u_angle
    flat = np.empty(2 * half)
    flat[:half] = rad * np.cos(ang)
    flat[half:] = rad * np.sin(ang)
    return flat[:count].reshape(rows, cols)


# ---------------------------------------------------------------------------
# Graph-side boundary (graph.py)
# ---------------------------------------------------------------------------

def mutual_knn_graph(vectors: np.ndarray, k: int, gamma: float, block: int = 1024) -> sp.csr_matrix:
    """Mutual k-NN adjacency (``graph.py:65-115``).

    Per row: clipped dots with self set to -inf then clipped to 0
    (``:96-98``), stable descending top-k so ties go to the lower column
    (``:58``), nonpositive sims dropped (``:61``), weights ``dot**gamma``
    (``:102``); the mutual graph is ``min(W, W^T)`` (``:111``).
    """
    n = vectors.shape[0]
    rows, cols, vals = [], [], []
    for s in range(0, n, block):
        e = min(n, s + block)
        sims = vectors[s:e] @ vectors.T
        sims[np.arange(e - s), np.arange(s, e)] = -np.inf
        np.maximum(sims, 0.0, out=sims)
        kk = min(k, n)
        top = np.argsort(-sims, axis=1, kind="stable")[:, :kk]
        rr = np.repeat(np.arange(e - s), kk)
        cc = top.ravel()
        ok = sims[rr, cc] > 0.0
        rows.append(rr[ok] + s)
        cols.append(cc[ok])
        vals.append(sims[rr[ok], cc[ok]] ** gamma)
    directed = sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                             shape=(n, n))
    mutual = directed.minimum(directed.T.tocsr())
    mutual.eliminate_zeros()
    mutual.sort_indices()
    return sp.csr_matrix(mutual)


def degrees(W: sp.csr_matrix) -> np.ndarray:
    """Row sums d = W 1 (``graph.py:118-121``)."""
    return np.asarray(W.sum(axis=1)).ravel()


def normalize_adjacency(W: sp.csr_matrix, deg: np.ndarray) -> sp.csr_matrix:
    """D^-1/2 W D^-1/2 with 0/0 = 0 (``graph.py:124-139``): entry
    ``(w_ij * s_i) * s_j`` with ``s = 1/sqrt(d)`` (0 where d = 0)."""
    s = np.zeros_like(deg, dtype=np.float64)
    pos = deg > 0
    s[pos] = 1.0 / np.sqrt(deg[pos])
    return sp.csr_matrix(W.multiply(s[:, None]).multiply(s[None, :]))


# ---------------------------------------------------------------------------
# Offline spectral path (spectral.py)
# ---------------------------------------------------------------------------

def range_finder(A: sp.csr_matrix, r_hat: int, q: int, seed: int, start: np.ndarray | None = None):
    """Simultaneous iteration (``spectral.py:147-171``): q x {Householder QR,
    re-QR when max|Q^T Q - I| > 1e-8, B = A Q}.  Returns (Q, B)."""
    n = A.shape[0]
    if not 1 <= r_hat <= n:
        raise ValueError("r_hat must lie in [1, n]")
    if q < 1:
        raise ValueError("q must be at least 1")
    Y = gaussian_matrix(n, r_hat, seed) if start is None else start
    Q = None
    for _ in range(q):
        Q = np.linalg.qr(Y)[0]
        if np.abs(Q.T @ Q - np.eye(r_hat)).max() > 1e-8:
            Q = np.linalg.qr(Q)[0]
        Y = A @ Q
    return Q, Y


def sign_fix(U: np.ndarray) -> np.ndarray:
    """Make the first largest-|u| entry of each column positive (``spectral.py:133-138``)."""
    lead = np.argmax(np.abs(U), axis=0)
    s = np.sign(U[lead, np.arange(U.shape[1])])
    s[s == 0] = 1.0
    return U * s


def row_norms(U) -> np.ndarray:
    """eta_i = ||U_i,:|| (``spectral.py:127-130``)."""
    if sp.issparse(U):
        return np.sqrt(np.asarray(U.multiply(U).sum(axis=1)).ravel())
    return np.linalg.norm(U, axis=1)


def rayleigh_ritz(Q: np.ndarray, B: np.ndarray, r: int):
    """C = Q^T B symmetrised, eigh, top r algebraically (stable), U = QV,
    sign fix, eta (``spectral.py:174-198``, ``_descending`` ``:141-144``)."""
    if not 1 <= r <= Q.shape[1]:
        raise ValueError("r out of range")
    C = Q.T @ B
    C = (C + C.T) / 2.0
    lam, V = np.linalg.eigh(C)
    pick = np.argsort(-lam, kind="stable")[:r]
    U = sign_fix(Q @ V[:, pick])
    return U, lam[pick], row_norms(U)


def decompose(A: sp.csr_matrix, r: int, p: int = 10, q: int = 4, seed: int = 0):
    """``spectral.py:297-309``: r_hat = min(r+p, n); range finder; Rayleigh-Ritz."""
    r_hat = min(r + p, A.shape[0])
    if r > r_hat:
        raise ValueError("r exceeds n")
    Q, B = range_finder(A, r_hat, q, seed)
    return rayleigh_ritz(Q, B, r)


def sparsify(U: np.ndarray, tau: int):
    """Keep exactly min(tau, nnz) entries of largest |u|, ties in (row, col)
    order (``spectral.py:269-294``).  Returns (U_tilde CSR, eta)."""
    if tau < 1:
        raise ValueError("tau must be positive")
    coo = sp.coo_matrix(U)
    keep = min(tau, coo.nnz)
    idx = np.lexsort((coo.col, coo.row, -np.abs(coo.data)))[:keep]
    Ut = sp.csr_matrix((coo.data[idx], (coo.row[idx], coo.col[idx])), shape=U.shape)
    Ut.sort_indices()
    return Ut, row_norms(Ut)


def sparsify_support(U: np.ndarray, tau: int) -> np.ndarray:
    """Sorted flat indices (row*r + col) of the entries ``sparsify`` keeps."""
    flat = np.abs(U).ravel()
    nz = np.flatnonzero(flat)
    keep = min(tau, nz.size)
    order = np.lexsort((nz, -flat[nz]))[:keep]
    return np.sort(nz[order])


# ---------------------------------------------------------------------------
# Online path (ranking.py)
# ---------------------------------------------------------------------------

def h_alpha(alpha: float):
    """(1-alpha)/(1-alpha x) (``ranking.py:45-65``)."""
    if not 0.0 <= alpha < 1.0:
        raise ValueError("alpha must lie in [0, 1)")
    return lambda x: (1.0 - alpha) / (1.0 - alpha * np.asarray(x, dtype=np.float64))


def heat_kernel(t: float):
    """exp(-t(1-x)), a nondecreasing custom transfer (BASELINE C5)."""
    return lambda x: np.exp(-t * (1.0 - np.asarray(x, dtype=np.float64)))


def transfer_values(h, lam: np.ndarray, analytic: bool = True) -> np.ndarray:
    """h(Lambda) with the 1024-point monotonicity probe for non-analytic h
    (``ranking.py:77-102``)."""
    if not analytic and lam.size and lam.max() > lam.min():
        grid = np.linspace(lam.min(), lam.max(), 1024)
        if np.any(np.diff(h(grid)) < -1e-12):
            raise ValueError("transfer function decreases on the spectrum")
    w = np.asarray(h(lam), dtype=np.float64)
    if not np.all(np.isfinite(w)):
        raise FloatingPointError("transfer function is not finite on the spectrum")
    return w


def filter_scores(U, lam: np.ndarray, eta: np.ndarray, w: np.ndarray,
                  y_idx: np.ndarray, y_val: np.ndarray, copy_uncovered: bool = True) -> np.ndarray:
    """x = U (w * U[supp y]^T y), then x_i := y_i on uncovered rows
    (eta_i == 0) of supp(y) (``ranking.py:219-255``)."""
    n, r = U.shape
    if y_idx.size == 0:
        z = np.zeros(r)
    else:
        rows = U[y_idx]
        z = np.asarray(rows.T @ y_val).ravel()
    x = np.asarray(U @ (w * z)).ravel()
    if copy_uncovered and y_idx.size:
        take = eta[y_idx] == 0.0
        if np.any(take):
            x[y_idx[take]] = y_val[take]
    return x


def neighbor_similarities(z: np.ndarray, data: np.ndarray, k: int, gamma: float) -> np.ndarray:
    """s(v_i | z) on the stable top-k of clipped dots, zeros dropped (``ranking.py:170-187``)."""
    sims = np.maximum(data @ z, 0.0)
    top = np.argsort(-sims, kind="stable")[:k]
    top = top[sims[top] > 0.0]
    out = np.zeros(data.shape[0])
    out[top] = sims[top] ** gamma
    return out


def observation_vector(regions: np.ndarray, data: np.ndarray, k: int, gamma: float, cap: int | None = None):
    """Sum of per-region neighbour similarities, stable top-cap, sorted indices
    (``ranking.py:190-216``).  Returns (indices int64, values float64)."""
    regions = np.atleast_2d(regions)
    cap = k if cap is None else cap
    y = np.zeros(data.shape[0])
    for reg in regions:
        y += neighbor_similarities(reg, data, k, gamma)
    top = np.argsort(-y, kind="stable")[:cap]
    top = top[y[top] > 0.0]
    if top.size == 0:
        warnings.warn("empty observation")
    top.sort()
    return top.astype(np.int64), y[top]


def rank(x: np.ndarray) -> np.ndarray:
    """Descending scores, ties by ascending index (``ranking.py:390-395``)."""
    return np.lexsort((np.arange(x.size), -x)).astype(np.int64)


# ---------------------------------------------------------------------------
# epilogues
# ---------------------------------------------------------------------------

def project(U, w, y_idx: np.ndarray, y_val: np.ndarray) -> np.ndarray:
    """w * U[supp y]^T y (``ranking.py:219-226`` scaled as in ``:244-246``)."""
    r = U.shape[1]
    if y_idx.size == 0:
        z = np.zeros(r)
    else:
        z = np.asarray(U[y_idx].T @ y_val).ravel()
    return z if w is None else w * z


def fsrw_correct(x: np.ndarray, eta: np.ndarray, vectors: np.ndarray, regions: np.ndarray) -> np.ndarray:
    """x + (1 - eta) * (V . sum of the query's region vectors) (``ranking.py:256-274``)."""
    regions = np.atleast_2d(regions)
    euclid = vectors @ regions.sum(axis=0)
    return np.asarray(x, dtype=np.float64) + (1.0 - eta) * euclid


def pooling_from_region_map(region_to_image: np.ndarray, n_images: int | None = None,
                            weights: np.ndarray | None = None) -> sp.csr_matrix:
    """(N, n) pooling CSR, one owning image per region (``ranking.py:300-311``)."""
    r2i = np.asarray(region_to_image, dtype=np.int64)
    n = r2i.size
    n_images = int(r2i.max()) + 1 if n_images is None else n_images
    data = np.ones(n) if weights is None else np.asarray(weights, dtype=np.float64)
    return sp.csr_matrix(sp.csr_matrix((data, (r2i, np.arange(n))), shape=(n_images, n)), dtype=np.float64)


def pool(P: sp.csr_matrix, x: np.ndarray) -> np.ndarray:
    """Image scores P x (``ranking.py:322-326``)."""
    return np.asarray(P @ np.asarray(x, dtype=np.float64)).ravel()


def pooled_basis(P: sp.csr_matrix, U) -> np.ndarray:
    """U_bar = P U as a dense (N, r) array (``ranking.py:329-334``)."""
    Ub = P @ U
    return Ub.toarray() if sp.issparse(Ub) else np.asarray(Ub)


def filter_pooled(U, w: np.ndarray, y_idx: np.ndarray, y_val: np.ndarray, U_bar: np.ndarray) -> np.ndarray:
    """U_bar (w * U[supp y]^T y), no uncovered copy (``ranking.py:337-353``)."""
    return U_bar @ project(U, w, y_idx, y_val)


def embedding(U, w: np.ndarray):
    """Phi = h(lam)^{1/2} U^T (``ranking.py:356-365``)."""
    if np.any(w < 0.0):
        raise ValueError("transfer values must be nonnegative to take a square root")
    scale = np.sqrt(w)
    if sp.issparse(U):
        return sp.diags(scale) @ U.T.tocsr()
    return scale[:, None] * U.T


def out_of_sample_similarity(z1: np.ndarray, z2: np.ndarray, phi, data: np.ndarray, k: int,
                             gamma: float) -> float:
    """(Phi psi(z1)) . (Phi psi(z2)), psi(z)_i = s(v_i | z) (``ranking.py:368-387``)."""
    e1 = np.asarray(phi @ neighbor_similarities(z1, data, k, gamma)).ravel()
    e2 = np.asarray(phi @ neighbor_similarities(z2, data, k, gamma)).ravel()
    return float(e1 @ e2)


# ---------------------------------------------------------------------------
# components and the blockwise decomposition
# ---------------------------------------------------------------------------

def mix_seed(seed: int, salt: int) -> int:
    """splitmix64 finalizer of (seed, salt) (``spectral.py:47-52``)."""
    z = (seed ^ ((salt + 1) * 0x9E3779B97F4A7C15)) & MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return (z ^ (z >> 31)) & MASK64


def connected_components(W: sp.csr_matrix):
    """(labels, sizes, order) by union-find, components by size desc then
    smallest vertex (``graph.py:215-250``)."""
    n = W.shape[0]
    parent = np.arange(n, dtype=np.int64)

    def find(i):
        root = i
        while parent[root] != root:
            root = parent[root]
        while parent[i] != root:
            parent[i], i = root, parent[i]
        return root

    coo = W.tocoo()
    for i, j in zip(coo.row.tolist(), coo.col.tolist()):
        if i < j:
            ri, rj = find(i), find(j)
            if ri != rj:
                parent[max(ri, rj)] = min(ri, rj)
    roots = np.array([find(i) for i in range(n)], dtype=np.int64)
    uniq, inverse, counts = np.unique(roots, return_inverse=True, return_counts=True)
    rank = np.lexsort((uniq, -counts))
    label_of = np.empty_like(rank)
    label_of[rank] = np.arange(rank.size)
    labels = label_of[inverse]
    return labels, counts[rank], np.argsort(labels, kind="stable")


def exact_eigenpairs(A: sp.csr_matrix, r: int | None = None):
    """Dense eigh, top r descending (stable), sign rule (``spectral.py:200-243``)."""
    vals, vecs = np.linalg.eigh(A.toarray())
    r = vals.size if r is None else r
    idx = np.argsort(-vals, kind="stable")[:r]
    U = sign_fix(vecs[:, idx])
    return U, vals[idx], row_norms(U)


def decompose_blockwise(A: sp.csr_matrix, labels: np.ndarray, r: int, rho: int, p: int = 10, q: int = 4,
                        seed: int = 0, dense_guard: int = 4096):
    """Per-component decomposition with a global top-r merge (``spectral.py:312-390``).
    Returns (U dense, eigenvalues, eta, all_exact, truncated)."""
    import math

    n = A.shape[0]
    blocks = []
    all_exact = True
    for comp in range(int(labels.max()) + 1):
        v = np.flatnonzero(labels == comp)
        sub = sp.csr_matrix(A[v][:, v])
        if v.size <= rho:
            U, lam, _ = exact_eigenpairs(sub)
        else:
            r_l = min(max(rho, math.ceil(r * v.size / n)), v.size)
            U, lam, _ = decompose(sub, r_l, p=p, q=q, seed=seed if comp == 0 else mix_seed(seed, comp))
            all_exact = False
        blocks.append((v, U, lam))
    lams = np.concatenate([b[2] for b in blocks])
    comps = np.concatenate([np.full(b[2].size, c) for c, b in enumerate(blocks)])
    cols = np.concatenate([np.arange(b[2].size) for b in blocks])
    keep = np.lexsort((cols, comps, -lams))[: min(r, lams.size)]
    U = np.zeros((n, keep.size))
    for out_col, cand in enumerate(keep):
        v, Ub, _ = blocks[comps[cand]]
        U[v, out_col] = Ub[:, cols[cand]]
    return U, lams[keep], row_norms(U), all_exact, keep.size < lams.size
