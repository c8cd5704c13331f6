"""Online step on a synthetic C3-shaped U~ through each certified path.

n = 1e6, r = 5000, ~100 entries per row (skewed lengths like the bench's U~),
b = 1024 k=50-sparse queries, top-100; times K9t ("tc"), K9h ("pruned") and
the unpruned path ("exact") with CUDA events (L2 flushed between steps) and
checks that all three return the same top-k bit for bit.

    python tools/online_paths_probe.py [--n 1000000 --r 5000 --per-row 100 --b 1024]
"""

import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1703_06935_b200 import _native as N  # noqa: E402
from paper_1703_06935_b200 import ranking, spectral  # noqa: E402
from paper_1703_06935_b200.graph import ComponentLabeling  # noqa: E402
from paper_1703_06935_b200.sparsemat import DeviceCSR  # noqa: E402


def synthetic_dec(n, r, per_row, dev, seed=5):
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    # lognormal row lengths (median ~ per_row / 2, long tail), capped at r
    lens = torch.exp(torch.randn(n, generator=g, device=dev) * 0.9) * per_row * 0.66
    lens = lens.clamp(0, r).to(torch.int64)
    indptr = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    indptr[1:] = torch.cumsum(lens, 0)
    nnz = int(indptr[-1])
    rows = torch.repeat_interleave(torch.arange(n, device=dev), lens)
    cols = torch.randint(0, r, (nnz,), generator=g, device=dev)
    key = rows * r + cols
    key = torch.unique(key)  # sorted, distinct (row, col)
    rows, cols = key // r, (key % r).to(torch.int32)
    counts = torch.bincount(rows, minlength=n)
    indptr[1:] = torch.cumsum(counts, 0)
    vals = (torch.randn(key.numel(), generator=g, device=dev) * 0.02).float()
    U = DeviceCSR(indptr, cols.contiguous(), vals, (n, r))
    eta = torch.zeros(n, dtype=torch.float64, device=dev)
    eta.index_add_(0, rows, vals.double() ** 2)
    lam = np.sort(np.random.default_rng(seed).uniform(-0.1, 0.7, r))[::-1].copy()
    return spectral.SpectralDecomposition(U, lam, eta.sqrt(), ComponentLabeling.trivial(n), spectral.Variant.SPARSE,
                                          spectral.Provenance(r=r, tau=key.numel(), seed=0))


def queries(n, b, k, seed=7):
    rng = np.random.default_rng(seed)
    ptr = [0]
    idx, val = [], []
    for _ in range(b):
        i = np.unique(rng.integers(0, n, size=k))
        idx.append(i)
        val.append(rng.random(i.size) ** 3 + 1e-3)
        ptr.append(ptr[-1] + i.size)
    return ranking.QueryBatch(n, np.asarray(ptr, np.int64), np.concatenate(idx), np.concatenate(val))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--r", type=int, default=5000)
    ap.add_argument("--per-row", type=int, default=100)
    ap.add_argument("--b", type=int, default=1024)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--paths", default="tc,pruned,exact")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    dec = synthetic_dec(a.n, a.r, a.per_row, dev)
    qb = queries(a.n, a.b, 50)
    dq = ranking.DeviceQueries(qb, torch.float32, dev)
    h = ranking.h_alpha(0.99)
    ctx = N.Context.get(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    t0 = time.perf_counter()
    ranking.dense_layout(dec)
    torch.cuda.synchronize()
    out = {"n": a.n, "r": a.r, "nnz": dec.U_device.nnz, "b": a.b, "dense_build_s": time.perf_counter() - t0}
    ref = None
    for path in a.paths.split(","):
        ctx.set_online_path(path)
        ctx.set_topk_prune(path != "exact")
        ws = torch.empty(ranking.filter_workspace_bytes(dec, a.b, want_x=False, topk=100), dtype=torch.uint8,
                         device=dev)
        res = ranking.FilterResult(top_idx=torch.empty(a.b, 100, dtype=torch.int64, device=dev),
                                   top_val=torch.empty(a.b, 100, dtype=torch.float32, device=dev))
        for _ in range(2):
            ranking.filter_device(dec, h, dq, topk=100, want_x=False, out=res, workspace=ws)
        torch.cuda.synchronize()
        ctx.enable_timing(True)
        ctx.stage_reset()
        ms = []
        for _ in range(a.steps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ranking.filter_device(dec, h, dq, topk=100, want_x=False, out=res, workspace=ws)
            e1.record()
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        st = {k: ctx.stage_time(k) for k in ("project", "filter_spmm", "copy_uncovered", "topk")}
        ctx.enable_timing(False)
        fb = ranking.last_fallback_count(ws, dec, a.b) if path != "exact" else 0
        extra = {}
        if ctx.last_online_path == "tc":
            st2 = ranking.last_tc_stats(ws, dec, a.b)
            extra = {"candidates_median": float(np.median(st2[:, 0])), "candidates_max": int(st2[:, 0].max()),
                     "rescored_median": float(np.median(st2[:, 1])), "rescored_max": int(st2[:, 1].max())}
        cur = (res.top_idx.cpu().numpy(), res.top_val.cpu().numpy())
        same = None
        if ref is not None:
            same = bool(np.array_equal(cur[0], ref[0]) and np.array_equal(cur[1].view(np.uint32), ref[1].view(np.uint32)))
        else:
            ref = cur
        out[path] = {"ms_per_step": float(np.median(ms)), "queries_per_s": a.b / (np.median(ms) / 1e3),
                     "stage_ms_per_step": {k: v[0] / a.steps for k, v in st.items()},
                     "fallback_queries": fb, "same_topk_as_first": same, "ran": ctx.last_online_path, **extra}
        del ws, res
        torch.cuda.empty_cache()
    ctx.set_topk_prune(True)
    ctx.set_online_path("tc")
    print(json.dumps(out))


if __name__ == "__main__":
    main()
