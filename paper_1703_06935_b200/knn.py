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
  product is 4e15 flops): a bf16 tensor-core GEMM (fp32 output) proposes
  kk = k + slack candidates per row, which are re-scored in the descriptors'
  dtype and ranked with the reference rule.  The selection is CERTIFIED:
  with e the rigorous bound on |x.y - s~| of the candidate GEMM
  (``score_error_bound``: bf16 rounding of both operands, 2u + u^2, plus the
  fp32 tensor-core accumulation, modelled per 16-element MMA step as in
  csrc/k9t.cu, times ||x|| max||y||) and m the kk-th largest approximate
  score, every vector left out scores at most m + e exactly; a row is
  certified when m + e < its k-th exact (clipped) score, or m + e <= 0 (the
  rest could only be zero-weight edges, which are dropped).  Rows that fail
  are recomputed with a split bf16x3 GEMM (x = hi + lo in bf16: hi.hi' +
  hi.lo' + lo.hi', error ~3u^2) and certified again; rows failing that too
  are scored by a GEMM in the descriptors' own dtype (the exact mode).
  The result equals the exact-dtype builder's graph (tests pin it against the
  reference's C1 and C2 graphs).
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
    return _candidates_scored(Ag @ Bg.T, kk, exclude_offset)[0]


def _candidates_scored(sims, kk, exclude_offset=None):
    """(top-kk indices, kk-th largest approximate score) per row of sims.

    On the device the selection is libfsr's exact top-k (fsr_topk_rows:
    sampled radix select + bitonic sort, (-x, index) order; ~10x faster than
    torch.topk on 2048 x 1e6 blocks)."""
    import torch

    from . import _native as N

    if exclude_offset is not None:
        ar = torch.arange(sims.shape[0], device=sims.device)
        sims[ar, ar + exclude_offset] = -float("inf")
    b, n = sims.shape
    if sims.is_cuda and sims.dtype in (torch.float32, torch.float64) and kk <= 1024 and sims.is_contiguous():
        idx = torch.empty(b, kk, dtype=torch.int64, device=sims.device)
        val = torch.empty(b, kk, dtype=sims.dtype, device=sims.device)
        N.Context.get(sims.device).call("topk_rows", N.dtype_code(sims.dtype), b, n, N.ptr(sims), n, kk, N.ptr(idx),
                                        N.ptr(val))
        return idx, val[:, kk - 1]
    top = torch.topk(sims, kk, dim=1, sorted=False)
    return top.indices, top.values.min(dim=1).values


BF16_U = 2.0 ** -8  # unit roundoff of bf16 (8-bit significand, round to nearest even)


def score_error_bound(d: int, scheme: str) -> float:
    """Rigorous bound on |x.y - s~| / (||x|| ||y||) for a candidate score s~.

    scheme "bf16": one bf16 GEMM with fp32 output: the rounded operands give
    |x y - bf(x) bf(y)| <= (2u + u^2) |x| |y| per product (products of two
    bf16 values are exact in fp32); the fp32 tensor-core accumulation loses
    at most 2^-20 of the running magnitude per 16-element MMA step (2x the
    model of csrc/k9t.cu, measured -2^-24 per step in tools/tc_debug.cu);
    Cauchy-Schwarz turns sum |x_l| |y_l| into ||x|| ||y||.
    scheme "bf16x3": x = hi + lo + dx with hi = bf(x), lo = bf(x - hi),
    |dx| <= u^2 |x|; s~ = hi.hi' + hi.lo' + lo.hi' misses lo.lo' and the dx
    terms (<= 3.1 u^2) and carries three accumulations plus two fp32 adds."""
    steps = -(-d // 16) + 1
    acc = steps * 2.0 ** -20
    u = BF16_U
    if scheme == "bf16":
        return 2 * u + u * u + acc * (1 + u) ** 2
    if scheme == "bf16x3":
        return 3.1 * u * u + 3 * acc * (1 + 2 * u) ** 2 + 2.0 ** -22
    raise ValueError(f"unknown scheme {scheme!r}")


def _approx_sims(A, X, scheme, split=None):
    """Candidate scores A @ X^T (fp32) by a bf16 GEMM or the split bf16x3 one.

    bf16x3 runs as ONE GEMM over a 3d-long K: [hi, hi, lo] . [hi', lo', hi']
    (split[2] holds the concatenated right operand): one fp32 accumulation
    of the three products per column instead of three outputs and two adds."""
    import torch

    bf = torch.bfloat16
    mm = lambda a, b: torch.mm(a, b.T, out_dtype=torch.float32)  # noqa: E731
    Ah = A.to(bf)
    Xh = X.to(bf) if split is None else split[0]
    if scheme == "bf16":
        return mm(Ah, Xh)
    Al = (A - Ah.to(A.dtype)).to(bf)
    if split is not None and len(split) > 2:
        return mm(torch.cat([Ah, Ah, Al], dim=1), split[2])
    Xl = (X - Xh.to(X.dtype)).to(bf) if split is None else split[1]
    return mm(Ah, Xh) + mm(Ah, Xl) + mm(Al, Xh)


def certified_topk(A, X, k: int, slack: int, exclude_offset=None, stats=None, split=None,
                   schemes=("bf16", "bf16x3", "exact")):
    """Per row of A: the k best columns of A X^T by (clipped score desc,
    index asc) and their exact clipped scores (A's dtype), from certified
    bf16 candidates (module doc).  Returns (indices, scores) (rows x k).
    ``schemes``: the certification stages to try in order ("exact" last)."""
    import torch

    n, d = X.shape
    kk = min(k + slack, n - (1 if exclude_offset is not None else 0))
    xmax = float(X.norm(dim=1).max())
    anorm = A.norm(dim=1)
    rows = torch.arange(A.shape[0], device=A.device)
    out_c = torch.empty(A.shape[0], k, dtype=torch.int64, device=A.device)
    out_v = torch.empty(A.shape[0], k, dtype=A.dtype, device=A.device)
    todo = rows
    for scheme in schemes:
        if todo.numel() == 0:
            break
        As = A[todo]
        if scheme == "exact":
            sims = As @ X.T
        else:
            sims = _approx_sims(As, X, scheme, split)
        if exclude_offset is not None:
            sims[torch.arange(todo.numel(), device=A.device), todo + exclude_offset] = -float("inf")
        cand, m = _candidates_scored(sims, kk)
        del sims
        exact = _rescore(As, X, cand)
        if exclude_offset is not None:
            exact[cand == (todo + exclude_offset)[:, None]] = 0.0
        c, v = _stable_topk(cand, exact, k)
        if scheme == "exact":
            ok = torch.ones(todo.numel(), dtype=torch.bool, device=A.device)
        else:
            e = score_error_bound(d, scheme) * anorm[todo].double() * xmax
            reach = m.double() + e
            ok = (reach < v[:, k - 1].double()) | (reach <= 0)
        done = todo[ok]
        out_c[done] = c[ok]
        out_v[done] = v[ok]
        if stats is not None:
            stats[scheme] = stats.get(scheme, 0) + int(ok.sum())
        todo = todo[~ok]
    return out_c, out_v


def _rescore(A, B, cand):
    """Exact clipped scores A[i] . B[cand[i, j]] in A's dtype."""
    import torch

    return torch.bmm(B[cand], A.unsqueeze(2)).squeeze(2).clamp_(min=0.0)


def mutual_knn_graph_device(X, k: int, gamma: float, block: int = 4096, slack: int = 16,
                            gemm_dtype=None, stats=None) -> SparseSymmetricMatrix:
    """Mutual k-NN adjacency of the rows of X (unit vectors) on the device.
    ``stats`` (a dict) receives how many rows each certification stage settled."""
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
    certified = gemm_dtype == torch.bfloat16 and X.dtype != torch.bfloat16
    if certified:
        block = min(block, 2048)  # fp32 candidate scores: block x n x 4 bytes
        hi = X.to(torch.bfloat16)
        lo = (X - hi.to(X.dtype)).to(torch.bfloat16)
        split = (hi, lo, torch.cat([hi, lo, hi], dim=1))  # the bf16x3 GEMM's K-concatenated operand
    schemes = ["bf16", "bf16x3", "exact"]
    for s in range(0, n, block):
        e = min(n, s + block)
        if certified:
            st = {}
            c, v = certified_topk(X[s:e], X, k, slack, exclude_offset=s, stats=st, split=split, schemes=schemes)
            if schemes[0] == "bf16" and st.get("bf16", 0) < (e - s) // 2:
                # the bf16 bound is too loose for these descriptors (e.g. d = 2048:
                # e ~ 0.008 against score gaps ~1e-3): start at bf16x3 from now on
                schemes = ["bf16x3", "exact"]
            if stats is not None:
                for key, v_ in st.items():
                    stats[key] = stats.get(key, 0) + v_
        else:
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
                             block: int = 1024, slack: int = 16, gemm_dtype=None, stats=None):
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
        if gemm_dtype == torch.bfloat16 and X.dtype != torch.bfloat16:
            c, v = certified_topk(R, X, k, slack, stats=stats)  # per region: k best, ties to the lower index
        else:
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
