"""Certified top-k pruning probe on the bench's real U~ (C3, 2%).

Question: if K9 gathers Zs rounded to fp16 (per-query power-of-two scale),
how many rows must be re-scored exactly so that the exact fp32 top-K is
provably among them?  For row i and query q,
  |x_i - x~_i| <= bound_i = sum_j |u_ij| |zs_j - zs~_j|  (+ fp32 rounding of both sums),
K-th largest exact >= T~ - L   (T~ = K-th largest x~, L = max bound over the x~ top-K),
so every exact top-K row satisfies x~_i + bound_i >= T~ - L: that set is re-scored.

    python tools/prune_probe.py [--queries 256] [--density 0.02]
"""

import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1703_06935_b200 import _native as N  # noqa: E402
from paper_1703_06935_b200 import ranking, spectral  # noqa: E402
from paper_1703_06935_b200.workloads import CONFIGS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--queries", type=int, default=256)
    ap.add_argument("--density", type=float, default=0.02)
    ap.add_argument("--K", type=int, default=100)
    a = ap.parse_args()
    cfg = CONFIGS["C3"]
    dev = torch.device("cuda", 0)
    b, K = a.queries, a.K
    S, (yp, yi, yv), _, _, _ = bench.build_inputs(cfg, cfg.n, b, dev, "float32")
    dec = spectral.decompose(S, cfg.r, p=cfg.p, q=cfg.q, seed=0, dtype="float32", device=dev)
    sd = spectral.sparsify(dec, int(round(a.density * cfg.n * cfg.r)))
    del dec
    torch.cuda.empty_cache()
    ctx = N.Context.get(dev)
    U = sd.U_device
    n, r = cfg.n, cfg.r
    w = ranking._weights_device(sd, ranking.h_alpha(cfg.alpha))
    q = ranking.DeviceQueries(ranking.QueryBatch(n, yp[:b + 1], yi[:yp[b]], yv[:yp[b]]), torch.float32, dev)
    Zt = torch.empty(b, r, device=dev)
    ctx.call("project_batch", N.F32, n, r, 1, N.ptr(U.indptr), N.ptr(U.indices), N.ptr(U.values), N.ptr(None), 0,
             N.ptr(w), b, N.ptr(q.y_ptr), N.ptr(q.y_idx), N.ptr(q.y_val), N.ptr(Zt))
    Zs = Zt.T.contiguous()  # r x b

    def spmm(vals, Z):
        Y = torch.empty(n, Z.shape[1], device=dev)
        ctx.call("csr_spmm", N.F32, n, N.ptr(U.indptr), N.ptr(U.indices), N.ptr(vals), Z.shape[1], N.ptr(Z),
                 Z.stride(0), N.ptr(Y), Y.stride(0))
        return Y

    X = spmm(U.values, Zs)
    true_tops = [torch.topk(X[:, j], K).indices for j in range(b)]
    rows_nnz = (U.indptr[1:] - U.indptr[:-1]).double()
    eta = sd.eta_device.double()  # row 2-norms of U~
    absU = U.values.abs().contiguous()
    amax = Zs.abs().amax(0).clamp_min(1e-30)
    zn = Zs.double().norm(dim=0)
    out = {"density": a.density, "queries": b, "K": K}
    for fmt in ("fp16", "bf16"):
        if fmt == "fp16":
            scale = torch.exp2(14 - torch.ceil(torch.log2(amax)))
            Zr = (Zs * scale).half().float() / scale
            rel_unit, sub = 2.0 ** -11, 2.0 ** -25 / scale.double()
        else:
            Zr = Zs.bfloat16().float()
            rel_unit, sub = 2.0 ** -8, torch.zeros_like(amax, dtype=torch.float64)
        Xr = spmm(U.values, Zr)
        exact_b = spmm(absU, (Zs - Zr).abs()).double()
        mag = spmm(absU, Zs.abs()).double()
        rnd = 2.0 * rows_nnz[:, None] * 2.0 ** -24 * mag
        # Cauchy-Schwarz bound: sum_j |u_ij||dz_j| <= rel * ||u_i|| ||zs_q|| (+ subnormal absolute part)
        cs = eta[:, None] * zn[None, :] * (rel_unit + 2.0 * rows_nnz[:, None] * 2.0 ** -24) * (1 + 1e-6) \
            + torch.sqrt(rows_nnz)[:, None] * eta[:, None] * sub[None, :]
        for name, bd in (("exact", exact_b * (1 + 1e-6) + rnd), ("cs", cs)):
            counts, missed = [], 0
            for j in range(b):
                xr = Xr[:, j].double()
                lower, upper = xr - bd[:, j], xr + bd[:, j]
                lam = torch.topk(lower, K).values[-1]
                cand = upper >= lam
                counts.append(int(cand.sum()))
                missed += int((~cand[true_tops[j]]).sum())
            c = np.array(counts)
            out[f"{fmt}_{name}"] = {"p50": float(np.percentile(c, 50)), "p90": float(np.percentile(c, 90)),
                                    "p99": float(np.percentile(c, 99)), "max": int(c.max()), "missed": missed}
        out[f"{fmt}_x_rel_l2_median"] = float(np.median([float((Xr[:, j] - X[:, j]).norm() / X[:, j].norm())
                                                        for j in range(b)]))
    print(json.dumps(out))


if __name__ == "__main__":
    main()
