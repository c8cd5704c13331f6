"""Distinct columns per 256-row tile of the bench's U~ (C3, 2%) under row
orders -- how much dense work a column-compacted tensor-core K9t could skip.

K9t multiplies every 256-row tile of the dense fp16 U~ with all r = 5000
columns of Zh.  If the rows of a tile only touch D << r distinct columns, a
tile-compacted layout (the tile's column list + a 256 x D dense block, Zh rows
gathered by TMA gather4) would do D / r of the MMA work.  Orders:

  natural   -- as generated (random w.r.t. clusters)
  dominant  -- rows sorted by the column of their largest |u| (then the second)
  label     -- rows sorted by the generator's cluster label (an oracle order)
  support   -- rows sorted by cluster label of ... (not available) -> omitted

    python tools/u_tile_probe.py
"""

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1703_06935_b200 import graph, knn, spectral, workloads  # noqa: E402
from paper_1703_06935_b200.workloads import CONFIGS  # noqa: E402


def tile_stats(indptr, indices, order, rows_per_tile, r, every=23):
    d = []
    n = order.numel()
    lens = indptr[1:] - indptr[:-1]
    for s in range(0, n - rows_per_tile + 1, rows_per_tile * every):
        rows = order[s:s + rows_per_tile]
        starts = indptr[:-1][rows]
        ln = lens[rows]
        off = torch.arange(int(ln.sum()), device=indices.device) - torch.repeat_interleave(
            torch.cumsum(ln, 0) - ln, ln)
        cols = indices[torch.repeat_interleave(starts, ln) + off]
        d.append(int(torch.unique(cols).numel()))
    d = np.asarray(d, dtype=np.float64)
    steps = np.ceil(d / 64.0) * 64.0
    return {"tiles_sampled": int(d.size), "distinct_mean": float(d.mean()), "distinct_p50": float(np.median(d)),
            "distinct_p90": float(np.percentile(d, 90)), "distinct_max": float(d.max()),
            "mma_work_fraction": float(steps.mean() / (np.ceil(r / 64.0) * 64.0))}


def main():
    cfg = CONFIGS["C3"]
    dev = torch.device("cuda", 0)
    n = cfg.n
    X, Qv, labels = workloads.device_cluster_descriptors(cfg, dev, n=n, queries=16)
    W = knn.mutual_knn_graph_device(X, cfg.k, cfg.gamma, gemm_dtype=torch.bfloat16)
    deg = graph.degrees_device(W, dev)
    S = graph.normalize_adjacency(W, deg, dtype="float32", device=dev)
    labels = labels[:n].clone()
    del X, Qv, W
    dec = spectral.decompose(S, cfg.r, p=cfg.p, q=cfg.q, seed=0, dtype="float32", device=dev)
    sd = spectral.sparsify(dec, int(round(cfg.density * n * cfg.r)))
    del dec
    torch.cuda.empty_cache()
    U = sd.U_device
    indptr, indices, vals = U.indptr, U.indices.long(), U.values
    lens = indptr[1:] - indptr[:-1]
    rows = torch.repeat_interleave(torch.arange(n, device=dev), lens)
    # dominant column per row: the column of the largest |u| (rows without entries: r)
    absv = vals.abs()
    mx = torch.zeros(n, device=dev).scatter_reduce_(0, rows, absv, "amax", include_self=True)
    is_max = absv >= mx[rows]
    dom = torch.full((n,), cfg.r, dtype=torch.int64, device=dev)
    dom.scatter_reduce_(0, rows[is_max], indices[is_max], "amin", include_self=True)
    # second key: the largest-|u| column among the rest (crudely: the first stored column)
    first = torch.where(lens > 0, indices[torch.clamp(indptr[:-1], max=indices.numel() - 1)],
                        torch.full_like(dom, cfg.r))
    orders = {
        "natural": torch.arange(n, device=dev),
        "dominant": torch.argsort(dom * (cfg.r + 1) + first),
        "label": torch.argsort(labels.long() * n + torch.arange(n, device=dev)),
        "label_then_dominant": torch.argsort((labels.long() * (cfg.r + 1) + dom) * 1),
    }
    out = {"n": n, "r": cfg.r, "nnz": int(U.nnz), "clusters": int(labels.max()) + 1}
    for name, order in orders.items():
        for rt in (128, 256):
            out[f"{name}_{rt}"] = tile_stats(indptr, indices, order, rt, cfg.r)
        print(json.dumps({name: {k: v for k, v in out.items() if k.startswith(name)}}), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
