"""K2 schedule microbenchmark: wide row panels vs L2-resident column panels.

A random CSR with the C3 graph's shape (n rows, nnz per row uniform in
[lo, hi], uniformly random columns -- no locality, like the mutual-kNN graph
of the synthetic clusters) times a dense n x k fp32 block.

    python tools/spmm_micro.py --n 1000000 --k 5500 [--panels 0,32,64,128]
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1703_06935_b200 import _native as N  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--k", type=int, default=5500)
    ap.add_argument("--lo", type=int, default=8)
    ap.add_argument("--hi", type=int, default=50)
    ap.add_argument("--panels", default="0,32,64,128")
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    ctx = N.Context.get(dev)
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    n, k = a.n, a.k
    deg = torch.randint(a.lo, a.hi + 1, (n,), generator=g, device=dev)
    indptr = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    indptr[1:] = torch.cumsum(deg, 0)
    nnz = int(indptr[-1])
    cols = torch.randint(0, n, (nnz,), generator=g, device=dev, dtype=torch.int32)
    # sort columns within rows (canonical CSR)
    rows = torch.repeat_interleave(torch.arange(n, device=dev), deg)
    key = rows * n + cols.long()
    cols = (torch.sort(key).values % n).to(torch.int32)
    vals = torch.rand(nnz, generator=g, device=dev)
    X = torch.randn(n, k, generator=g, device=dev)
    Y = torch.empty(n, k, device=dev)
    ref = None
    out = {"n": n, "k": k, "nnz": nnz, "gather_bytes": nnz * k * 4,
           "algorithmic_bytes": 8 * nnz + 8 * (n + 1) + 2 * 4 * n * k}
    for p in [int(x) for x in a.panels.split(",")]:
        ctx.set_spmm_panel(p)

        def run():
            ctx.call("csr_spmm", N.F32, n, N.ptr(indptr), N.ptr(cols), N.ptr(vals), k, N.ptr(X), k, N.ptr(Y), k)

        run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        if ref is None:
            ref = Y.clone()
            same = True
        else:
            same = bool(torch.equal(ref, Y))
        out[f"panel_{p}"] = {"ms": ms, "algorithmic_gbs": out["algorithmic_bytes"] / ms / 1e6,
                             "gather_gbs": out["gather_bytes"] / ms / 1e6, "bitwise_equal_to_first": same}
        print(json.dumps({p: out[f"panel_{p}"]}), flush=True)
    # One panel stored contiguously (n x w): what a panel-major copy of X would give.
    del X, Y, ref
    for w in (8, 16, 32):
        Xc = torch.randn(n, w, generator=g, device=dev)
        Yc = torch.empty(n, w, device=dev)
        ctx.set_spmm_panel(w * 4)

        def runc():
            ctx.call("csr_spmm", N.F32, n, N.ptr(indptr), N.ptr(cols), N.ptr(vals), w, N.ptr(Xc), w, N.ptr(Yc), w)

        runc()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            runc()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        out[f"contig_{w}"] = {"ms_per_pass": ms, "extrapolated_ms": ms * k / w}
        print(json.dumps({f"contig_{w}": out[f"contig_{w}"]}), flush=True)
    ctx.set_spmm_panel(0)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
