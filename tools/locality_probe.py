"""Probe: does a locality permutation of the vertices speed up K2 / K9?

Builds the C2 (or --config) inputs like bench.py, then times
  * K2 (S x Q, r_hat columns) in the as-generated order and after a reverse
    Cuthill-McKee permutation of the vertices;
  * K9 (U~ x Zs, b columns) with U~'s rows in both orders;
and prints structure statistics (distinct columns per row block of U~).
"""

import argparse
import json
import os
import sys
import time

import numpy as np
import scipy.sparse as sp
from scipy.sparse.csgraph import reverse_cuthill_mckee

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from bench import build_inputs  # noqa: E402
from paper_1703_06935_b200 import _native as N  # noqa: E402
from paper_1703_06935_b200 import spectral  # noqa: E402
from paper_1703_06935_b200.sparsemat import DeviceCSR  # noqa: E402
from paper_1703_06935_b200.workloads import CONFIGS  # noqa: E402


def time_spmm(ctx, A: DeviceCSR, X, reps=5):
    Y = torch.empty(A.shape[0], X.shape[1], dtype=X.dtype, device=X.device)
    spectral._spmm(ctx, N.dtype_code(X.dtype), A, X, Y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        spectral._spmm(ctx, N.dtype_code(X.dtype), A, X, Y)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, Y


def permute_csr(csr: sp.csr_matrix, perm_rows, perm_cols=None):
    out = csr[perm_rows]
    if perm_cols is not None:
        out = out[:, perm_cols]
    out = sp.csr_matrix(out)
    out.sort_indices()
    return out


def block_distinct_cols(csr, block):
    n = csr.shape[0]
    tot, cnt = 0, 0
    for s in range(0, n - block, max(block, n // 2000)):
        cols = csr.indices[csr.indptr[s]:csr.indptr[s + block]]
        tot += np.unique(cols).size
        cnt += 1
    return tot / max(cnt, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--b", type=int, default=1024)
    a = ap.parse_args()
    cfg = CONFIGS[a.config]
    n = a.n or cfg.n
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    S, _, t_in, nnz_w, iso = build_inputs(cfg, n, 64, dev, "float32")
    ctx = N.Context.get(dev)
    r_hat = cfg.r + cfg.p
    out = {"n": n, "nnz": S.nnz, "inputs_s": t_in}
    Sd = S.device(torch.float32, dev)
    Q = spectral.gaussian_block(n, r_hat, 0, dtype="float32", device=dev)
    t_orig, Y0 = time_spmm(ctx, Sd, Q)
    Sh = Sd.to_scipy()
    t0 = time.perf_counter()
    perm = reverse_cuthill_mckee(Sh, symmetric_mode=True).astype(np.int64)
    out["rcm_s"] = time.perf_counter() - t0
    Sp = permute_csr(Sh, perm, perm)
    Spd = DeviceCSR.from_scipy(Sp, torch.float32, dev)
    Qp = Q[torch.as_tensor(perm, device=dev)].contiguous()
    t_rcm, Yp = time_spmm(ctx, Spd, Qp)
    err = (Yp - Y0[torch.as_tensor(perm, device=dev)]).abs().max().item()
    bw = lambda csr: float(np.abs(np.repeat(np.arange(csr.shape[0]), np.diff(csr.indptr)) - csr.indices).mean())
    out.update(k2_ms_orig=t_orig, k2_ms_rcm=t_rcm, k2_check=err, mean_abs_i_minus_j_orig=bw(Sh),
               mean_abs_i_minus_j_rcm=bw(Sp))
    es = 4
    bytes_k2 = S.nnz * 8 + (n + 1) * 8 + 2 * es * n * r_hat
    out["k2_gbs_orig"] = bytes_k2 / t_orig / 1e6
    out["k2_gbs_rcm"] = bytes_k2 / t_rcm / 1e6
    # decomposition in both orders -> U~ structure and K9 time
    dec = spectral.decompose(S, cfg.r, p=cfg.p, q=cfg.q, dtype="float32", device=dev)
    sdec = spectral.sparsify(dec, cfg.tau if n == cfg.n else int(cfg.density * n * cfg.r))
    del dec
    U = sdec.U_device.to_scipy()
    rn = np.diff(U.indptr)
    out["u_row_nnz_pct"] = {p: float(np.percentile(rn, p)) for p in (0, 10, 50, 90, 99, 100)}
    out["u_rows_empty"] = int((rn == 0).sum())
    Up = permute_csr(U, perm)
    for blk in (32, 128):
        out[f"u_distinct_cols_per_{blk}_orig"] = block_distinct_cols(U, blk)
        out[f"u_distinct_cols_per_{blk}_rcm"] = block_distinct_cols(Up, blk)
    # order rows by their largest-|u| column (eigenvector "home")
    home = np.array([U.indices[U.indptr[i] + np.argmax(np.abs(U.data[U.indptr[i]:U.indptr[i + 1]]))]
                     if rn[i] else -1 for i in range(n)])
    ph = np.argsort(home, kind="stable")
    Uh = permute_csr(U, ph)
    for blk in (32, 128):
        out[f"u_distinct_cols_per_{blk}_home"] = block_distinct_cols(Uh, blk)
    Zs = torch.randn(cfg.r, a.b, device=dev)
    for name, M in (("orig", U), ("rcm", Up), ("home", Uh)):
        Md = DeviceCSR.from_scipy(M, torch.float32, dev)
        t, _ = time_spmm(ctx, Md, Zs)
        out[f"k9_ms_{name}"] = t
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
