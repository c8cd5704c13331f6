"""Could a single query skip rows by Cauchy-Schwarz?  |x_i| <= ||u_i|| ||w.z||,
so rows with ||u_i|| ||w.z|| < t (t = the query's 100th largest score) cannot
reach its top-100.  On the bench's C3 decomposition (2% U~) this reports, per
query, the fraction of rows (and of U~'s entries) that survive that test --
what a norm-sorted U~ layout would still have to stream for b = 1."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1703_06935_b200 import ranking, spectral  # noqa: E402
from paper_1703_06935_b200.workloads import CONFIGS  # noqa: E402


def main():
    cfg = CONFIGS["C3"]
    dev = torch.device("cuda", 0)
    S, (yp, yi, yv), _, _, _ = bench.build_inputs(cfg, cfg.n, 64, dev, "float32")
    dec = spectral.decompose(S, cfg.r, p=cfg.p, q=cfg.q, seed=0, dtype="float32", device=dev)
    sd = spectral.sparsify(dec, int(round(0.02 * cfg.n * cfg.r)))
    del dec
    U = sd.U_device
    eta = sd.eta_device.float()
    lens = (U.indptr[1:] - U.indptr[:-1]).float()
    h = ranking.h_alpha(0.99)
    w = ranking._weights_device(sd, h)
    qb = ranking.QueryBatch(cfg.n, yp, yi, yv)
    dq = ranking.DeviceQueries(qb, sd.dtype, dev)
    X = ranking.filter_device(sd, h, dq).X  # 64 x n exact scores
    Zt = ranking._project_device(sd, w, dq)  # 64 x r scaled projections
    out = []
    for j in range(X.shape[0]):
        t = torch.topk(X[j], 100).values[-1].item()
        zn = Zt[j].norm().item()
        keep = eta * zn >= t
        out.append({"t": t, "zs_norm": zn, "rows_frac": keep.float().mean().item(),
                    "entries_frac": (lens[keep].sum() / lens.sum()).item()})
    rows = np.array([o["rows_frac"] for o in out])
    ents = np.array([o["entries_frac"] for o in out])
    print(json.dumps({"queries": len(out), "rows_frac_median": float(np.median(rows)), "rows_frac_max": float(rows.max()),
                      "entries_frac_median": float(np.median(ents)), "entries_frac_max": float(ents.max()),
                      "first": out[:4]}))


if __name__ == "__main__":
    main()
