"""b=1 online latency on the bench's real U~ (C3) at 1/2/5% density: K9
(SpMV) device time over many repetitions (FSR_SPMV_PIPE selected kernel
variants while they were being compared; see spmm.cuh).

    python tools/b1_probe.py [--reps 50]
"""

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_1703_06935_b200 import _native as N  # noqa: E402
from paper_1703_06935_b200 import ranking, spectral  # noqa: E402
from paper_1703_06935_b200.workloads import CONFIGS  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=50)
    a = ap.parse_args()
    cfg = CONFIGS["C3"]
    dev = torch.device("cuda", 0)
    S, (yp, yi, yv), _, _, _ = bench.build_inputs(cfg, cfg.n, 64, dev, "float32")
    dec = spectral.decompose(S, cfg.r, p=cfg.p, q=cfg.q, seed=0, dtype="float32", device=dev)
    batch = ranking.QueryBatch(cfg.n, yp, yi, yv)
    h = ranking.h_alpha(0.99)
    ctx = N.Context.get(dev)
    out = {}
    for d in (0.01, 0.02, 0.05):
        sd = spectral.sparsify(dec, int(round(d * cfg.n * cfg.r)))
        q1 = ranking.DeviceQueries(ranking.QueryBatch(cfg.n, yp[:2], yi[: yp[1]], yv[: yp[1]]), sd.dtype, dev)
        res = ranking.FilterResult()
        ws = None
        for var in ("0",) * 3:
            os.environ["FSR_SPMV_PIPE"] = var
            for _ in range(3):
                ranking.filter_device(sd, h, q1, topk=100, want_x=False, out=res)
            torch.cuda.synchronize()
            ctx.enable_timing(True)
            ctx.stage_reset()
            for _ in range(a.reps):
                ranking.filter_device(sd, h, q1, topk=100, want_x=False, out=res)
            torch.cuda.synchronize()
            ms, cnt = ctx.stage_time("filter_spmm")
            ctx.enable_timing(False)
            out.setdefault(f"{d}", {}).setdefault(f"pipe{var}", []).append(round(ms / cnt, 4))
        del sd
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
