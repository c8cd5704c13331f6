"""Structure of the bench's U~ (C3): row-length skew and column sharing
between rows, to size the reuse a row-reordered K9 could get.

    python tools/u_structure_probe.py [--n 1000000]
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1703_06935_b200 import spectral  # noqa: E402
from paper_1703_06935_b200.workloads import CONFIGS  # noqa: E402


def block_reuse(indptr, indices, order, rows_per_block):
    """mean over blocks of (nnz in block) / (distinct columns in block), rows taken in `order`."""
    n = order.size
    tot_nnz, tot_distinct = 0, 0
    for s in range(0, n - rows_per_block + 1, rows_per_block * 97):  # sample every 97th block
        rows = order[s:s + rows_per_block]
        cols = np.concatenate([indices[indptr[r]:indptr[r + 1]] for r in rows])
        tot_nnz += cols.size
        tot_distinct += np.unique(cols).size
    return tot_nnz / max(tot_distinct, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=None)
    a = ap.parse_args()
    cfg = CONFIGS["C3"]
    n = a.n or cfg.n
    dev = torch.device("cuda", 0)
    S, _, _, _, _ = bench.build_inputs(cfg, n, 64, dev, "float32")
    dec = spectral.decompose(S, cfg.r, p=cfg.p, q=cfg.q, seed=0, dtype="float32", device=dev)
    sdec = spectral.sparsify(dec, int(round(cfg.density * n * cfg.r)))
    U = sdec.U_device
    indptr = U.indptr.cpu().numpy()
    indices = U.indices.cpu().numpy()
    lens = np.diff(indptr)
    out = {"n": n, "nnz": int(indptr[-1]),
           "row_len_pct": {p: float(np.percentile(lens, p)) for p in (0, 10, 50, 90, 99, 99.9, 100)},
           "empty_rows": int((lens == 0).sum())}
    srt = np.sort(lens)[::-1]
    cum = np.cumsum(srt)
    out["rows_holding_50pct_nnz"] = int(np.searchsorted(cum, cum[-1] * 0.5)) + 1
    out["rows_holding_90pct_nnz"] = int(np.searchsorted(cum, cum[-1] * 0.9)) + 1
    first = np.where(lens > 0, indices[np.minimum(indptr[:-1], indices.size - 1)], -1)
    second = np.where(lens > 1, indices[np.minimum(indptr[:-1] + 1, indices.size - 1)], -1)
    natural = np.arange(n)
    by_first = np.lexsort((second, first))
    for rb in (32, 128):
        out[f"reuse_natural_{rb}"] = block_reuse(indptr, indices, natural, rb)
        out[f"reuse_sorted_first_cols_{rb}"] = block_reuse(indptr, indices, by_first, rb)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
