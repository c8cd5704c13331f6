"""Dense-stage microbenchmark at C3 shapes: Gram, cross, apply (B R^-1), lift.

    python tools/dense_micro.py --n 1000000 --k 5500 --r 5000 [--path auto|cublas]
"""

import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1703_06935_b200 import _native as N  # noqa: E402


def timed(fn, reps=2):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--k", type=int, default=5500)
    ap.add_argument("--r", type=int, default=5000)
    ap.add_argument("--path", default="auto")
    ap.add_argument("--only", default="gram,cross,apply,lift")
    ap.add_argument("--apply-slices", type=int, default=4, help="R^-1 slices in apply (1 = first CholQR pass)")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    ctx = N.Context.get(dev)
    ctx.set_dense_path(a.path)
    n, k, r = a.n, a.k, a.r
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    Q = torch.randn(n, k, generator=g, device=dev) / np.sqrt(n)
    B = torch.randn(n, k, generator=g, device=dev) / np.sqrt(n)
    G = torch.empty(k, k, dtype=torch.float64, device=dev)
    out = {"n": n, "k": k, "r": r, "path": a.path}
    only = a.only.split(",")
    if "gram" in only:
        ms = timed(lambda: ctx.call("gram", N.F32, n, k, N.ptr(Q), k, N.ptr(G), 0))
        out["gram_ms"] = ms
        out["gram_useful_tflops"] = n * k * k / (ms * 1e-3) / 1e12  # symmetric half: n k^2 flops
    if "cross" in only:
        ms = timed(lambda: ctx.call("cross", N.F32, n, k, N.ptr(Q), k, N.ptr(B), k, N.ptr(G), 0))
        out["cross_ms"] = ms
        out["cross_tflops"] = 2 * n * k * k / (ms * 1e-3) / 1e12
    if "apply" in only:
        Gs = (Q[:20000].double().T @ Q[:20000].double())
        Gs += torch.eye(k, dtype=torch.float64, device=dev) * 0.1
        R = torch.linalg.cholesky(Gs).T.contiguous()  # upper
        Rc = R.T.contiguous()  # column-major storage of R
        Bw = B.clone()
        ms = timed(lambda: ctx.call("apply_rinv_levels", N.F32, n, k, N.ptr(Rc), N.ptr(Bw), k, a.apply_slices),
                   reps=1)
        out["apply_slices"] = a.apply_slices
        out["apply_ms"] = ms
        out["apply_tflops"] = 2 * n * k * k / (ms * 1e-3) / 1e12
        del Bw
    if "lift" in only:
        V = torch.randn(k, r, dtype=torch.float64, device=dev, generator=g)
        U = torch.empty(n, r, device=dev)
        ms = timed(lambda: ctx.call("lift", N.F32, n, k, r, N.ptr(Q), k, N.ptr(V), N.ptr(U), r))
        out["lift_ms"] = ms
        out["lift_tflops"] = 2 * n * k * r / (ms * 1e-3) / 1e12
    print(json.dumps(out))


if __name__ == "__main__":
    main()
