"""K9t selection statistics per transfer function on the bench's C3 2% U~ (b = 1024):
candidates per query, rows re-scored, fallback queries, stage times.

    python tools/tf_stats_probe.py
"""

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_1703_06935_b200 import _native as N  # noqa: E402
from paper_1703_06935_b200 import ranking, spectral  # noqa: E402
from paper_1703_06935_b200.workloads import CONFIGS  # noqa: E402


def main():
    cfg = CONFIGS["C3"]
    dev = torch.device("cuda", 0)
    ctx = N.Context.get(dev)
    b = 1024
    S, (y_ptr, y_idx, y_val), _, _, _ = bench.build_inputs(cfg, cfg.n, b, dev, "float32")
    dec = spectral.decompose(S, cfg.r, p=cfg.p, q=cfg.q, seed=0, dtype="float32", device=dev)
    sd = spectral.sparsify(dec, int(round(0.02 * cfg.n * cfg.r)))
    del dec
    torch.cuda.empty_cache()
    qb = ranking.QueryBatch(cfg.n, y_ptr, y_idx, y_val)
    dq = ranking.DeviceQueries(qb, sd.dtype, dev)
    ws = torch.empty(ranking.filter_workspace_bytes(sd, b, want_x=False, topk=100), dtype=torch.uint8, device=dev)
    flush = bench.L2Flush(dev)
    ctx.enable_timing(True)
    for name, h in (("h_alpha(0.99)", ranking.h_alpha(0.99)), ("h_alpha(0.9)", ranking.h_alpha(0.9)),
                    ("heat(10)", ranking.heat_kernel(10.0))):
        res = ranking.FilterResult()
        for _ in range(3):
            ranking.filter_device(sd, h, dq, topk=100, want_x=False, out=res, workspace=ws)
        torch.cuda.synchronize()
        ctx.stage_reset()
        for _ in range(5):
            flush()
            ranking.filter_device(sd, h, dq, topk=100, want_x=False, out=res, workspace=ws)
        torch.cuda.synchronize()
        st = ranking.last_tc_stats(ws, sd, b)
        stages = {k: ctx.stage_time(k)[0] / 5 for k in ("project", "filter_spmm", "topk")}
        w = ranking.transfer_values(h, sd.eigenvalues)
        print(json.dumps({"h": name, "path": ctx.last_online_path, "stage_ms": stages,
                          "candidates": {"median": float(np.median(st[:, 0])), "p90": float(np.percentile(st[:, 0], 90)),
                                         "max": int(st[:, 0].max())},
                          "rescored": {"median": float(np.median(st[:, 1])), "max": int(st[:, 1].max())},
                          "fallback_queries": ranking.last_fallback_count(ws, sd, b),
                          "w_min_max": [float(w.min()), float(w.max())]}), flush=True)


if __name__ == "__main__":
    main()
