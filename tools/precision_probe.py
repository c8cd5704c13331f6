"""Which dense stage limits fp32-mode accuracy?  C1 golden, stage-wise path switch.

For each combination of (range finder path, Rayleigh-Ritz path) in
{auto (int8 Ozaki), cublas}, run fp32 decompose on the C1 golden graph and
report Ritz error (normwise) and x rel-L2 vs the reference fixtures.
"""

import json
import os
import sys

import numpy as np
import scipy.sparse as sp

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import torch  # noqa: E402

from paper_1703_06935_b200 import _native as N  # noqa: E402
from paper_1703_06935_b200 import ranking, spectral  # noqa: E402
from paper_1703_06935_b200.sparsemat import SparseSymmetricMatrix  # noqa: E402


def main():
    g = dict(np.load(os.path.join(REPO, "tests", "golden", "c1.npz")))
    n, r, p, q, tau, seed = (int(v) for v in g["params"])
    S = SparseSymmetricMatrix(sp.csr_matrix((g["S_data"], g["W_indices"], g["W_indptr"]), shape=(n, n)))
    batch = ranking.QueryBatch(n, g["y_ptr"], g["y_idx"], g["y_val"])
    h = ranking.h_alpha(float(g["alpha"]))
    ctx = N.Context.get()
    out = []
    fast_opts = [True, False]
    for rf in ("auto", "cublas"):
        for rr in ("auto", "cublas"):
            for fast in fast_opts:
                spectral.FAST_FIRST_GRAM = fast
                spectral.FAST_FIRST_APPLY = fast
                ctx.set_dense_path(rf)
                basis = spectral.range_finder(S, r + p, q, seed, dtype="float32")
                Qd = basis.Q.double().cpu().numpy()
                orth = float(np.abs(Qd.T @ Qd - np.eye(r + p)).max())
                ctx.set_dense_path(rr)
                dec = spectral.approx_eigendecomposition(S, basis, r)
                ctx.set_dense_path("auto")
                lam_err = float(np.abs(dec.eigenvalues - g["lam"]).max() / np.abs(g["lam"]).max())
                X = ranking.filter_batch(dec, h, batch)
                xa = g["x_approx"]
                xerr = [float(np.linalg.norm(X[j] - xa[j]) / np.linalg.norm(xa[j])) for j in range(xa.shape[0])]
                out.append({"range_finder": rf, "rayleigh_ritz": rr, "fast_first_gram": fast, "orth": orth,
                            "ritz_err": lam_err, "x_err_max": max(xerr), "x_err_median": float(np.median(xerr))})
                print(json.dumps(out[-1]), flush=True)
    spectral.FAST_FIRST_GRAM = True
    spectral.FAST_FIRST_APPLY = True


if __name__ == "__main__":
    main()
