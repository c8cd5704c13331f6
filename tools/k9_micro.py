"""K9 (online filter SpMM) microbenchmark on a synthetic C3-shaped U~.

U~: n x r CSR with `per_row` random sorted columns per row (tau = n*per_row),
fp32 values; Zs comes from a real K8 projection of b random 50-sparse
queries.  Runs fsr_filter_batch (X materialised, top-100) and reports the
per-stage device times from libfsr's stage timers, plus an fp64 check of a
few queries.

    python tools/k9_micro.py [--b 1024] [--runs 2]
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
    ap.add_argument("--r", type=int, default=5000)
    ap.add_argument("--per-row", type=int, default=100)
    ap.add_argument("--b", type=int, default=1024)
    ap.add_argument("--runs", type=int, default=1)
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    ctx = N.Context.get(dev)
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    n, r, b = a.n, a.r, a.b
    tau = n * a.per_row
    indptr = torch.arange(0, tau + 1, a.per_row, dtype=torch.int64, device=dev)
    # canonical CSR (sorted, distinct columns per row): stratified random columns
    stride = r // a.per_row
    cols = (torch.arange(a.per_row, device=dev, dtype=torch.int32) * stride
            + torch.randint(0, stride, (n, a.per_row), generator=g, device=dev, dtype=torch.int32))
    cols = cols.reshape(-1).contiguous()
    vals = (torch.randn(tau, generator=g, device=dev) * 1e-3).contiguous()
    w = torch.rand(r, generator=g, device=dev)
    eta = torch.ones(n, dtype=torch.float64, device=dev)
    y_ptr = torch.arange(0, 50 * b + 1, 50, dtype=torch.int64, device=dev)
    ys = n // 50
    y_idx = (torch.arange(50, device=dev) * ys + torch.randint(0, ys, (b, 50), generator=g, device=dev)).reshape(-1)
    y_val = torch.rand(50 * b, generator=g, device=dev)
    X = torch.empty(b, n, device=dev)
    topk = 100
    ti = torch.empty(b, topk, dtype=torch.int64, device=dev)
    tv = torch.empty(b, topk, device=dev)
    need = int(ctx.lib.fsr_filter_workspace_bytes(N.F32, n, r, b, 0))
    ws = torch.empty(need, dtype=torch.uint8, device=dev)

    def run():
        ctx.call("filter_batch", N.F32, n, r, 1, N.ptr(indptr), N.ptr(cols), N.ptr(vals), N.ptr(None), 0, N.ptr(w),
                 N.ptr(eta), b, N.ptr(y_ptr), N.ptr(y_idx), N.ptr(y_val), 1, N.ptr(ws), N.ptr(X), topk, N.ptr(ti),
                 N.ptr(tv))

    # fp64 check of a few queries (plain torch index_add on the device)
    check_j = [0, b // 2, b - 1]

    def check():
        errs = []
        for j in check_j:
            s, e = j * 50, (j + 1) * 50
            rows = y_idx[s:e]
            z = torch.zeros(r, dtype=torch.float64, device=dev)
            for t in range(50):
                i = int(rows[t])
                p0, p1 = int(indptr[i]), int(indptr[i + 1])
                z.index_add_(0, cols[p0:p1].long(), vals[p0:p1].double() * float(y_val[s + t]))
            zs = z * w.double()
            x = torch.zeros(n, dtype=torch.float64, device=dev)
            rr = torch.repeat_interleave(torch.arange(n, device=dev), a.per_row)
            x.index_add_(0, rr, vals.double() * zs[cols.long()])
            errs.append(float((X[j].double() - x).norm() / x.norm()))
        return max(errs)

    ref = None
    res = {"n": n, "r": r, "tau": tau, "b": b}
    variants = os.environ.get("MICRO_VARIANTS", "").split(",") if os.environ.get("MICRO_VARIANTS") else [None]
    for v in range(a.runs * len(variants)):
        if variants[0] is not None:
            os.environ[os.environ.get("MICRO_VARIANT_ENV", "FSR_SPMV_VARIANT")] = variants[v % len(variants)]
        run()
        torch.cuda.synchronize()
        ctx.enable_timing(True)
        ctx.stage_reset()
        for _ in range(a.reps):
            run()
        torch.cuda.synchronize()
        ms = ctx.stage_time("filter_spmm")[0] / a.reps
        ctx.enable_timing(False)
        if ref is None:
            ref = X.clone()
        err = float((X - ref).abs().max() / ref.abs().max())
        out = {"run": v, "variant": variants[v % len(variants)], "check_rel_l2": check(), "k9_ms": ms, "tflops": 2 * tau * b / ms / 1e9,
               "l2_gather_tbs": 4 * tau * b / ms / 1e9, "max_rel_diff_vs_first": err}
        res[f"run{v}"] = out
        print(json.dumps(out), flush=True)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
