"""Head/tail eigen-split probe on the bench's U~ (C3, 2%): x_i = sum over the first J
columns (computed) + the rest (bounded by ||u_i,tail||_2 ||zs_tail||_2); how many rows
would have to be re-scored for the top-100.  Result: the synthetic spectrum is flat,
so the tail bound keeps nearly every row (profiles/r01/headtail_probe.json).

    python tools/headtail_probe.py
"""
import os, sys, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import bench
from paper_1703_06935_b200 import _native as N, ranking, spectral
from paper_1703_06935_b200.workloads import CONFIGS
cfg = CONFIGS["C3"]
dev = torch.device("cuda", 0)
b = 128
S, (yp, yi, yv), _, _, _ = bench.build_inputs(cfg, cfg.n, b, dev, "float32")
dec = spectral.decompose(S, cfg.r, p=cfg.p, q=cfg.q, seed=0, dtype="float32", device=dev)
sd = spectral.sparsify(dec, int(round(0.02 * cfg.n * cfg.r)))
del dec, S; torch.cuda.empty_cache()
lam = sd.eigenvalues
out = {"lam_quantiles": {str(p): float(np.percentile(lam, p)) for p in (0, 10, 50, 90, 99, 100)}}
h = ranking.h_alpha(cfg.alpha)
w = ranking.transfer_values(h, lam)
out["w_first"] = [float(x) for x in w[[0, 10, 100, 250, 500, 1000, 2000, 4999]]]
ctx = N.Context.get(dev)
U = sd.U_device
n, r = cfg.n, cfg.r
wd = torch.as_tensor(w, dtype=torch.float32, device=dev)
q = ranking.DeviceQueries(ranking.QueryBatch(n, yp[:b + 1], yi[:yp[b]], yv[:yp[b]]), torch.float32, dev)
Zt = torch.empty(b, r, device=dev)
ctx.call("project_batch", N.F32, n, r, 1, N.ptr(U.indptr), N.ptr(U.indices), N.ptr(U.values), N.ptr(None), 0,
         N.ptr(wd), b, N.ptr(q.y_ptr), N.ptr(q.y_idx), N.ptr(q.y_val), N.ptr(Zt))
Zs = Zt.T.contiguous()
def spmm(vals, Z):
    Y = torch.empty(n, Z.shape[1], device=dev)
    ctx.call("csr_spmm", N.F32, n, N.ptr(U.indptr), N.ptr(U.indices), N.ptr(vals), Z.shape[1], N.ptr(Z), Z.stride(0), N.ptr(Y), Y.stride(0))
    return Y
X = spmm(U.values, Zs)
rows = torch.repeat_interleave(torch.arange(n, device=dev), U.indptr[1:] - U.indptr[:-1])
cols = U.indices.long()
K = 100
for J in (50, 100, 250, 500, 1000, 2000):
    head = cols < J
    vh = torch.where(head, U.values, torch.zeros_like(U.values)).contiguous()
    H = spmm(vh, Zs)
    rho = torch.zeros(n, device=dev, dtype=torch.float64).index_add_(0, rows, torch.where(head, 0.0, U.values.double() ** 2)).sqrt()
    zt = Zs[J:].double().norm(dim=0)  # per query
    cnts, missed = [], 0
    for j in range(b):
        bd = rho * zt[j] * (1 + 1e-6) + 1e-7 * X[:, j].abs().double().max()
        hj = H[:, j].double()
        lam_k = torch.topk(hj - bd, K).values[-1]
        cand = (hj + bd) >= lam_k
        cnts.append(int(cand.sum()))
        missed += int((~cand[torch.topk(X[:, j], K).indices]).sum())
    c = np.array(cnts)
    out[f"J{J}"] = {"head_entry_frac": float(head.float().mean()), "zs_tail_over_total_median": float(np.median((zt / Zs.double().norm(dim=0)).cpu().numpy())),
                    "cand_p50": float(np.median(c)), "cand_p90": float(np.percentile(c, 90)), "cand_max": int(c.max()), "missed": missed}
    print(json.dumps({f"J{J}": out[f"J{J}"]}), flush=True)
print(json.dumps(out))
