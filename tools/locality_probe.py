"""Column locality of the bench's U~ (C3, 2%) under row orderings.

K9h gathers one 512-byte fp16 Zs segment per entry of U~; rows of one CTA
(32) or one SM (4 CTAs) that share columns could hit L1 instead of L2.  For a
few row orders this reports 1 - distinct(block, col) / nnz, the idealised
fraction of gathers an L1 holding the block's segments would serve.

    python tools/locality_probe.py
"""

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1703_06935_b200 import spectral  # noqa: E402
from paper_1703_06935_b200.workloads import CONFIGS  # noqa: E402


def main():
    cfg = CONFIGS["C3"]
    dev = torch.device("cuda", 0)
    S, _, _, _, _ = bench.build_inputs(cfg, cfg.n, 256, dev, "float32")
    dec = spectral.decompose(S, cfg.r, p=cfg.p, q=cfg.q, seed=0, dtype="float32", device=dev)
    sd = spectral.sparsify(dec, int(round(0.02 * cfg.n * cfg.r)))
    del dec
    U = sd.U_device
    n, r = cfg.n, cfg.r
    lens = (U.indptr[1:] - U.indptr[:-1])
    rows = torch.repeat_interleave(torch.arange(n, device=dev), lens)
    cols = U.indices.long()
    a = U.values.abs()
    # dominant column of each row (largest |u|); rows with no entries -> r
    dom = torch.full((n,), r, dtype=torch.long, device=dev)
    best = torch.full((n,), -1.0, device=dev)
    best.scatter_reduce_(0, rows, a, "amax")
    hit = a == best[rows]
    dom.scatter_reduce_(0, rows[hit], cols[hit], "amin", include_self=True)
    orders = {"index": torch.arange(n, device=dev),
              "dominant_col": torch.argsort(dom * (n + 1) + torch.arange(n, device=dev))}
    out = {"n": n, "r": r, "nnz": int(U.nnz), "points": []}
    for name, perm in orders.items():
        pos = torch.empty_like(perm)
        pos[perm] = torch.arange(n, device=dev)
        for B in (32, 128, 1024):
            key = (pos[rows] // B) * r + cols
            d = torch.unique(key).numel()
            pt = {"order": name, "block_rows": B, "reuse": 1 - d / cols.numel()}
            out["points"].append(pt)
            print(json.dumps(pt), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
