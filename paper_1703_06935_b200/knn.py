"""Device-side builders for the inputs of the hot path (synthetic workloads).

``mutual_knn_graph_device`` produces the mutual k-NN adjacency W of
reference ``graph.py:65-115`` for descriptor sets far beyond what the CPU
reference can build (n = 1e6: days on the host).  Candidates
come from a bf16 similarity GEMM (k + slack per row), are re-scored exactly in
fp32 and ranked with the reference's tie rule (descending similarity, lower
index first, self excluded, zero similarities dropped); W = min(W, W^T) keeps
mutual edges only, weights s^gamma.  This is input generation for the bench --
SURVEY.md 8(f) ranks a fully exact GPU kNN builder as the next row.

``observation_batch_device`` builds k-sparse query signals y with values
[q^T v]_+^gamma on the top-k similarities (BASELINE C5; reference
``ranking.py:170-216`` for a single region).
"""

from __future__ import annotations

import numpy as np

from .sparsemat import DeviceCSR, SparseSymmetricMatrix


def _stable_topk(cand, sims, k):
    """Per row: the k best (sim desc, index asc) among candidate columns."""
    import torch

    idx_order = torch.argsort(cand, dim=1)
    cand = torch.gather(cand, 1, idx_order)
    sims = torch.gather(sims, 1, idx_order)
    order = torch.argsort(-sims, dim=1, stable=True)[:, :k]
    return torch.gather(cand, 1, order), torch.gather(sims, 1, order)


def mutual_knn_graph_device(X, k: int, gamma: float, block: int = 4096, slack: int = 16,
                            gemm_dtype=None) -> SparseSymmetricMatrix:
    import torch

    n, d = X.shape
    if k < 1 or k >= n:
        raise ValueError("k must lie in [1, n)")
    gemm_dtype = gemm_dtype or torch.bfloat16
    Xg = X.to(gemm_dtype)
    kk = min(k + slack, n - 1)
    nbr = torch.empty(n, k, dtype=torch.int64, device=X.device)
    val = torch.empty(n, k, dtype=torch.float32, device=X.device)
    for s in range(0, n, block):
        e = min(n, s + block)
        sims = Xg[s:e] @ Xg.T
        ar = torch.arange(e - s, device=X.device)
        sims[ar, ar + s] = -float("inf")
        cand = torch.topk(sims, kk, dim=1, sorted=False).indices
        del sims
        exact = torch.bmm(X[cand], X[s:e].unsqueeze(2)).squeeze(2).clamp_(min=0.0)
        exact[cand == (ar + s)[:, None]] = -1.0  # never self
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


def observation_batch_device(Qv, X, k: int, gamma: float, block: int = 1024):
    """k-sparse y per query row of Qv: top-k of [q^T v]_+ (stable), values ^gamma,
    indices sorted, zeros dropped.  Returns host (y_ptr, y_idx, y_val)."""
    import torch

    b = Qv.shape[0]
    idx_all, val_all = [], []
    for s in range(0, b, block):
        e = min(b, s + block)
        sims = (Qv[s:e] @ X.T).clamp_(min=0.0)
        top = torch.topk(sims, k, dim=1)
        idx_all.append(top.indices)
        val_all.append(top.values)
    idx = torch.cat(idx_all).cpu().numpy()
    val = torch.cat(val_all).double().cpu().numpy() ** gamma
    ptr = [0]
    out_i, out_v = [], []
    for j in range(b):
        ok = val[j] > 0
        ii, vv = idx[j][ok], val[j][ok]
        o = np.argsort(ii)
        out_i.append(ii[o])
        out_v.append(vv[o])
        ptr.append(ptr[-1] + ii.size)
    return np.asarray(ptr, np.int64), np.concatenate(out_i).astype(np.int64), np.concatenate(out_v)
