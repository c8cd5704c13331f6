"""K2 (B = W Q) on the C3 graph under vertex orderings.

K2 gathers one 1 KB row segment of Q per nonzero per 256-column panel and
sweeps the rows in order, panel by panel.  If a row's neighbours sit within
~100k positions of it (100 MB of a 256-column fp32 panel = L2), the gathers
hit L2 instead of DRAM.  This probe relabels the C3 graph's vertices
(new row i = old row perm[i], each row's entries kept in their original
order, columns renamed) and times K2 for:

  index  -- the generated order (random w.r.t. clusters)
  rcm    -- reverse Cuthill-McKee of W's pattern (scipy.sparse.csgraph)
  label  -- sorted by the generator's cluster label (an oracle order: the
            best cluster locality the data can offer; not available to a user)

It checks Y_perm == Y[perm] bit for bit (same per-row sums) and reports the
neighbour-distance profile of each order.

    python tools/k2_order_probe.py [--n 1000000] [--k 5500]
"""

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1703_06935_b200 import _native as N  # noqa: E402
from paper_1703_06935_b200 import graph, knn, workloads  # noqa: E402
from paper_1703_06935_b200.workloads import CONFIGS  # noqa: E402


def permute_csr(indptr, indices, vals, perm):
    """Relabel: new row i = old row perm[i]; entries in their original order."""
    dev = indptr.device
    n = perm.numel()
    pos = torch.empty_like(perm)
    pos[perm] = torch.arange(n, device=dev)
    lens = (indptr[1:] - indptr[:-1])[perm]
    ip = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    ip[1:] = torch.cumsum(lens, 0)
    starts = torch.repeat_interleave(indptr[:-1][perm], lens)
    off = torch.arange(int(ip[-1]), device=dev) - torch.repeat_interleave(ip[:-1], lens)
    src = starts + off
    return ip, pos[indices[src].long()].to(torch.int32), vals[src], pos


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--k", type=int, default=5500)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--orders", default="index,rcm,label")
    ap.add_argument("--panels", default="0")
    ap.add_argument("--contig", type=int, default=256,
                    help="also time K2 over Q stored panel-major ([panel][n][w], w columns); 0 = off")
    a = ap.parse_args()
    cfg = CONFIGS["C3"]
    n = a.n or cfg.n
    dev = torch.device("cuda", 0)
    ctx = N.Context.get(dev)
    t0 = time.perf_counter()
    X, Qv, labels = workloads.device_cluster_descriptors(cfg, dev, n=n, queries=16)
    W = knn.mutual_knn_graph_device(X, cfg.k, cfg.gamma, gemm_dtype=torch.bfloat16)
    deg = graph.degrees_device(W, dev)
    S = graph.normalize_adjacency(W, deg, dtype="float32", device=dev)
    labels = labels[:n].clone()
    del X, Qv
    A = S.device(torch.float32, dev)
    indptr, indices, vals = A.indptr, A.indices, A.values
    nnz = int(indices.numel())
    out = {"n": n, "k": a.k, "nnz": nnz, "inputs_s": time.perf_counter() - t0,
           "algorithmic_bytes": 8 * nnz + 8 * (n + 1) + 2 * 4 * n * a.k, "gather_bytes": nnz * a.k * 4, "orders": {}}
    print(json.dumps({k: v for k, v in out.items() if k != "orders"}), flush=True)
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    Q = torch.randn(n, a.k, generator=g, device=dev)
    Y = torch.empty_like(Q)
    rows = torch.repeat_interleave(torch.arange(n, device=dev), indptr[1:] - indptr[:-1])

    def k2(ip, ix, vv, Qm, Ym, w=None):
        w = w or a.k
        ctx.call("csr_spmm", N.F32, n, N.ptr(ip), N.ptr(ix), N.ptr(vv), w, N.ptr(Qm), w, N.ptr(Ym), w)

    def timed(ip, ix, vv, Qm, Ym):
        k2(ip, ix, vv, Qm, Ym)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            k2(ip, ix, vv, Qm, Ym)
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / a.reps

    ctx.set_spmm_panel(0)
    k2(indptr, indices, vals, Q, Y)
    torch.cuda.synchronize()
    for name in a.orders.split(","):
        t1 = time.perf_counter()
        if name == "index":
            perm = torch.arange(n, device=dev)
        elif name == "rcm":
            import scipy.sparse as sp
            from scipy.sparse.csgraph import reverse_cuthill_mckee

            m = sp.csr_matrix((np.ones(nnz, np.int8), indices.cpu().numpy(), indptr.cpu().numpy()), shape=(n, n))
            perm = torch.as_tensor(reverse_cuthill_mckee(m, symmetric_mode=True).astype(np.int64), device=dev)
        elif name == "label":
            perm = torch.argsort(labels * n + torch.arange(n, device=dev))
        else:
            raise SystemExit(f"unknown order {name}")
        order_s = time.perf_counter() - t1
        ip, ix, vv, pos = permute_csr(indptr, indices, vals, perm)
        dist = (pos[rows] - pos[indices.long()]).abs().float()
        prof = {"order_s": order_s, "mean_abs_i_minus_j": float(dist.mean()),
                "median_abs_i_minus_j": float(dist.median()),
                "frac_within_10k": float((dist < 1e4).float().mean()),
                "frac_within_100k": float((dist < 1e5).float().mean())}
        del dist
        Qp = Q[perm]
        Yp = torch.empty_like(Qp)
        for p in [int(x) for x in a.panels.split(",")]:
            ctx.set_spmm_panel(p)
            ms = timed(ip, ix, vv, Qp, Yp)
            prof[f"panel_{p}"] = {"ms": ms, "algorithmic_gbs": out["algorithmic_bytes"] / ms / 1e6,
                                  "gather_gbs": out["gather_bytes"] / ms / 1e6,
                                  "bitwise_equal_to_index_order": bool(torch.equal(Yp, Y[perm]))}
        ctx.set_spmm_panel(0)
        if a.contig:
            # Q panel-major: each w-column panel of Q contiguous (n x w); one K2 launch per panel
            w = a.contig
            P = -(-a.k // w)
            Qc = torch.zeros(P, n, w, device=dev)
            for p in range(P):
                c1 = min(a.k, (p + 1) * w)
                Qc[p, :, :c1 - p * w] = Qp[:, p * w:c1]
            Yc = torch.empty(n, w, device=dev)
            for p in range(P):
                k2(ip, ix, vv, Qc[p], Yc, w)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.reps):
                for p in range(P):
                    k2(ip, ix, vv, Qc[p], Yc, w)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / a.reps
            c0 = (P - 1) * w
            same = bool(torch.equal(Yc[:, :a.k - c0], Yp[:, c0:]))
            t0_ = torch.cuda.Event(enable_timing=True)
            t1_ = torch.cuda.Event(enable_timing=True)
            t0_.record()
            for p in range(P):
                c1 = min(a.k, (p + 1) * w)
                Qc[p, :, :c1 - p * w] = Qp[:, p * w:c1]
            t1_.record()
            torch.cuda.synchronize()
            prof[f"contig_{w}"] = {"ms": ms, "algorithmic_gbs": out["algorithmic_bytes"] / ms / 1e6,
                                   "gather_gbs": out["gather_bytes"] / ms / 1e6,
                                   "last_panel_bitwise_equal": same,
                                   "panel_major_copy_ms (torch, not optimised)": t0_.elapsed_time(t1_)}
            del Qc, Yc
        out["orders"][name] = prof
        print(json.dumps({name: prof}), flush=True)
        del Qp, Yp, ip, ix, vv, pos
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
