"""Device builders for the inputs of the hot path: the mutual k-NN graph W and
the observation vectors Y.

``mutual_knn_graph_device`` follows reference ``graph.py:49-115``
(``build_mutual_knn_graph`` + ``_top_k_rows``): per row, the k most similar
other vectors by (clipped similarity descending, column ascending), edges with
similarity 0 dropped, weight max(v_i.v_j, 0)**gamma, and W = min(W, W^T) so
only mutual edges survive (the two directed weights of a pair can differ in
the last bit; the minimum is kept, as scipy's ``minimum`` does).

``observation_batch_device`` follows ``ranking.py:168-216``
(``neighbor_similarities`` + ``observation_vector``): for every region of a
query, the k best dataset vectors by (clipped dot descending, index
ascending) contribute sim**gamma; regions are summed in order; the sum is cut
to the ``cap`` largest entries (same tie rule), zeros dropped, indices sorted.

Both use a candidate GEMM followed by an exact re-score:

* ``gemm_dtype`` = the descriptors' dtype (default): candidates and scores
  come from the same product, so the selection is exact for that dtype.  With
  float64 descriptors this is the parity mode (tests pin it against the
  reference's own C1 graph and query vectors).
* ``gemm_dtype=torch.bfloat16`` (C3/C4 bench inputs, n = 1e6: the n^2 d
  product is 4e15 flops): a bf16 tensor-core GEMM proposes k + slack
  candidates per row, which are re-scored in the descriptors' dtype and
  ranked with the reference rule.  A true neighbour can be missed only if its
  bf16 score falls below slack other candidates (bf16 dot error ~1e-4).
"""

from __future__ import annotations

import numpy as np

from .sparsemat import DeviceCSR, SparseSymmetricMatrix


def _stable_topk(cand, sims, k):
    """Per row: the k best candidates by (sim desc, index asc)."""
    import torch

    idx_order = torch.argsort(cand, dim=1)
    cand = torch.gather(cand, 1, idx_order)
    sims = torch.gather(sims, 1, idx_order)
    order = torch.argsort(-sims, dim=1, stable=True)[:, :k]
    return torch.gather(cand, 1, order), torch.gather(sims, 1, order)


def _candidates(Ag, Bg, kk, exclude_offset=None):
    """Top-kk column candidates of Ag @ Bg^T per row (self excluded if offset given)."""
    import torch

    sims = Ag @ Bg.T
    if exclude_offset is not None:
        ar = torch.arange(Ag.shape[0], device=Ag.device)
        sims[ar, ar + exclude_offset] = -float("inf")
    return torch.topk(sims, kk, dim=1, sorted=False).indices


def _rescore(A, B, cand):
    """Exact clipped scores A[i] . B[cand[i, j]] in A's dtype."""
    import torch

    return torch.bmm(B[cand], A.unsqueeze(2)).squeeze(2).clamp_(min=0.0)


def mutual_knn_graph_device(X, k: int, gamma: float, block: int = 4096, slack: int = 16,
                            gemm_dtype=None) -> SparseSymmetricMatrix:
    """Mutual k-NN adjacency of the rows of X (unit vectors) on the device."""
    import torch

    n, d = X.shape
    if gamma <= 0:
        raise ValueError("gamma must be positive")
    if k < 1:
        raise ValueError("k must be positive")
    if k >= n:
        raise ValueError(f"k must be smaller than the number of vectors ({k} >= {n})")
    gemm_dtype = gemm_dtype or X.dtype
    Xg = X if gemm_dtype == X.dtype else X.to(gemm_dtype)
    kk = min(k + slack, n - 1)
    nbr = torch.empty(n, k, dtype=torch.int64, device=X.device)
    val = torch.empty(n, k, dtype=X.dtype, device=X.device)
    for s in range(0, n, block):
        e = min(n, s + block)
        cand = _candidates(Xg[s:e], Xg, kk, exclude_offset=s)
        exact = _rescore(X[s:e], X, cand)
        exact[cand == torch.arange(s, e, device=X.device)[:, None]] = 0.0  # self scores 0 (dropped below)
        c, v = _stable_topk(cand, exact, k)
        nbr[s:e] = c
        val[s:e] = v
    rows = torch.arange(n, device=X.device).repeat_interleave(k)
    cols = nbr.reshape(-1)
    w = val.reshape(-1)
    keep = w > 0.0
    rows, cols, w = rows[keep], cols[keep], w[keep].double() ** gamma
    key = rows * n + cols
    key, perm = torch.sort(key)
    w = w[perm]
    rev = (key % n) * n + key // n
    pos = torch.searchsorted(key, rev).clamp_(max=key.numel() - 1)
    mutual = key[pos] == rev
    wmin = torch.minimum(w, w[pos])
    key, w = key[mutual], wmin[mutual]
    r_ = key // n
    c_ = (key % n).to(torch.int32)
    counts = torch.bincount(r_, minlength=n)
    indptr = torch.zeros(n + 1, dtype=torch.int64, device=X.device)
    indptr[1:] = torch.cumsum(counts, 0)
    return SparseSymmetricMatrix.from_device(DeviceCSR(indptr, c_, w.contiguous(), (n, n)))


def observation_batch_device(Qv, X, k: int, gamma: float, cap: int | None = None, regions: int = 1,
                             block: int = 1024, slack: int = 16, gemm_dtype=None):
    """Observation vectors of b queries with ``regions`` region vectors each.

    Qv: (b * regions, d) unit rows, the regions of query j at rows
    [j * regions, (j + 1) * regions).  Returns host CSC arrays
    (y_ptr, y_idx int64 sorted per query, y_val float64).
    """
    import torch

    if k < 1 or k > X.shape[0]:
        raise ValueError(f"k must lie in [1, n], got {k}")
    if gamma <= 0:
        raise ValueError("gamma must be positive")
    cap = k if cap is None else cap
    if cap < 1:
        raise ValueError("cap must be positive")
    if Qv.shape[0] % regions:
        raise ValueError("query rows must be a multiple of regions")
    n = X.shape[0]
    b = Qv.shape[0] // regions
    gemm_dtype = gemm_dtype or X.dtype
    Xg = X if gemm_dtype == X.dtype else X.to(gemm_dtype)
    kk = min(k + slack, n)
    ck = min(cap + slack, n)
    qblk = max(1, block // regions)
    out_i, out_v, ptr = [], [], [0]
    for s in range(0, b, qblk):
        e = min(b, s + qblk)
        R = Qv[s * regions:e * regions]
        cand = _candidates(R.to(gemm_dtype), Xg, kk)
        exact = _rescore(R, X, cand)
        c, v = _stable_topk(cand, exact, k)          # per region: k best, ties to the lower index
        v = torch.where(v > 0, v.double() ** gamma, torch.zeros_like(v, dtype=torch.float64))
        y = torch.zeros(e - s, n, dtype=torch.float64, device=X.device)
        for t in range(regions):                      # regions summed in order (ranking.py:208-209)
            rows = torch.arange(e - s, device=X.device)[:, None].expand(-1, k)
            y.index_put_((rows.reshape(-1), c[t::regions].reshape(-1)), v[t::regions].reshape(-1), accumulate=True)
        top = torch.topk(y, ck, dim=1, sorted=False)
        ci, cv = _stable_topk(top.indices, top.values, cap)
        for j in range(e - s):
            ok = cv[j] > 0
            ii, vv = ci[j][ok], cv[j][ok]
            o = torch.argsort(ii)
            out_i.append(ii[o].cpu().numpy())
            out_v.append(vv[o].cpu().numpy())
            ptr.append(ptr[-1] + int(ok.sum()))
    return (np.asarray(ptr, np.int64), np.concatenate(out_i).astype(np.int64),
            np.concatenate(out_v).astype(np.float64))
