"""Online-path microbenchmark on a synthetic U~ (no graph / decomposition).

    python tools/online_micro.py --n 1000000 --r 5000 --nnz 100 --skew 0 --b 1

Builds a random CSR U~ (n x r, `nnz` per row on average; --skew > 0 draws row
lengths from a lognormal), random eigenvalues, k=50-sparse queries, and times
filter_device (top-100) per stage.
"""

import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1703_06935_b200 import _native as N  # noqa: E402
from paper_1703_06935_b200 import ranking, spectral  # noqa: E402
from paper_1703_06935_b200.graph import ComponentLabeling  # noqa: E402
from paper_1703_06935_b200.sparsemat import DeviceCSR  # noqa: E402


def synth(n, r, nnz, skew, dev, seed=0):
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    if skew > 0:
        lens = torch.exp(torch.randn(n, generator=g, device=dev) * skew)
        lens = (lens / lens.mean() * nnz).round().clamp_(0, r).long()
    else:
        lens = torch.full((n,), nnz, dtype=torch.long, device=dev)
    indptr = torch.zeros(n + 1, dtype=torch.long, device=dev)
    indptr[1:] = torch.cumsum(lens, 0)
    tot = int(indptr[-1])
    cols = torch.randint(0, r, (tot,), generator=g, device=dev, dtype=torch.int32)
    # canonical CSR (sorted, distinct columns per row): key = row * r + col, deduplicated
    rows = torch.repeat_interleave(torch.arange(n, device=dev), lens)
    key = torch.unique(rows * r + cols.long())  # sorted
    rows = key // r
    cols = (key % r).to(torch.int32)
    indptr = torch.zeros(n + 1, dtype=torch.long, device=dev)
    indptr[1:] = torch.cumsum(torch.bincount(rows, minlength=n), 0)
    tot = int(key.numel())
    vals = torch.randn(tot, generator=g, device=dev) / np.sqrt(nnz)
    return DeviceCSR(indptr, cols, vals.float(), (n, r))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--r", type=int, default=5000)
    ap.add_argument("--nnz", type=int, default=100)
    ap.add_argument("--skew", type=float, default=0.0)
    ap.add_argument("--b", type=int, nargs="+", default=[1, 64, 1024])
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--prune", default="on", choices=["on", "off", "both"],
                    help="top-k-only batches through the certified pruned path (on), the unpruned fp32 K9 (off), "
                         "or both (and check they agree)")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    U = synth(a.n, a.r, a.nnz, a.skew, dev)
    lam = np.sort(np.random.default_rng(1).uniform(-0.2, 1.0, a.r))[::-1].copy()
    eta = torch.ones(a.n, dtype=torch.float64, device=dev)
    dec = spectral.SpectralDecomposition(U, lam, eta, ComponentLabeling.trivial(a.n), spectral.Variant.SPARSE,
                                         spectral.Provenance())
    ctx = N.Context.get(dev)
    ctx.enable_timing(True)
    rng = np.random.default_rng(2)
    h = ranking.h_alpha(0.99)
    out = {"n": a.n, "r": a.r, "nnz": U.nnz, "skew": a.skew, "points": []}
    modes = {"on": [True], "off": [False], "both": [True, False]}[a.prune]
    batches = {}
    for b in a.b:
        ptr = np.arange(b + 1, dtype=np.int64) * 50
        idx = np.concatenate([np.sort(rng.choice(a.n, 50, replace=False)) for _ in range(b)])
        batches[b] = ranking.QueryBatch(a.n, ptr, idx, rng.random(b * 50) ** 3)
    for b, prune in [(b, p) for b in a.b for p in modes]:
        ctx.set_topk_prune(prune)
        qb = batches[b]
        dq = ranking.DeviceQueries(qb, torch.float32, dev)
        res = ranking.FilterResult()
        for _ in range(3):
            ranking.filter_device(dec, h, dq, topk=100, want_x=False, out=res)
        torch.cuda.synchronize()
        ctx.stage_reset()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            ranking.filter_device(dec, h, dq, topk=100, want_x=False, out=res)
        e1.record()
        torch.cuda.synchronize()
        st = {k: ctx.stage_time(k)[0] / a.reps for k in ("project", "filter_spmm", "copy_uncovered", "topk")}
        ms = e0.elapsed_time(e1) / a.reps
        bytes_k9 = U.nnz * 8 + (a.n + 1) * 8 + 4 * a.r * b + 4 * a.n * b
        pt = {"b": b, "prune": prune, "variant": os.environ.get("FSR_K9H_VARIANT", "0"), "ms": ms,
              "qps": b / ms * 1e3, "stages_ms": st, "k9_gbs": bytes_k9 / (st["filter_spmm"] * 1e-3) / 1e9}
        if a.prune == "both":
            top = (res.top_idx.cpu(), res.top_val.cpu())
            if prune:
                first = top
            else:
                pt["identical_to_pruned"] = bool(torch.equal(first[0], top[0]) and
                                                 torch.equal(first[1].view(torch.int32), top[1].view(torch.int32)))
        out["points"].append(pt)
        print(json.dumps(pt), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
