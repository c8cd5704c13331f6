"""Small-batch online step (K9s) on the bench's C3 decomposition.

Builds the C3 inputs and the 2% U~ exactly as bench.py does, then times the
certified top-100 step for b in {1, 8, 64} (eager filter_device and one
FilterGraph replay), per stage (libfsr CUDA events), and wraps five b = 1
graph replays in the NVTX range "k9s:b1" for ncu launch lists / captures:

    python tools/stream_probe.py [--density 0.02]
    ncu --nvtx --nvtx-include "k9s:b1/" --metrics gpu__time_duration.sum ... python tools/stream_probe.py
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
    ap.add_argument("--density", type=float, default=0.02)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--batches", default="1,8,64")
    ap.add_argument("--topk-segs", type=int, default=0, help="FSR_OPT_TOPK_SEGMENTS (0 = automatic)")
    ap.add_argument("--single", default=None, help="b = 1 path: sell (K9e) | csr")
    ap.add_argument("--sell-long", type=int, default=0, help="ranking.SELL_LONG_ROW override")
    ap.add_argument("--sell-share", type=float, default=0.0, help="ranking.SELL_MAX_LONG_SHARE override")
    a = ap.parse_args()
    cfg = CONFIGS["C3"]
    dev = torch.device("cuda", 0)
    ctx = N.Context.get(dev)
    ctx.set_topk_segments(a.topk_segs)
    if a.single:
        ctx.single_query_path = a.single
    if a.sell_long:
        ranking.SELL_LONG_ROW = a.sell_long
    if a.sell_share:
        ranking.SELL_MAX_LONG_SHARE = a.sell_share
    S, (y_ptr, y_idx, y_val), _, _, _ = bench.build_inputs(cfg, cfg.n, 256, dev, "float32")
    dec = spectral.decompose(S, cfg.r, p=cfg.p, q=cfg.q, seed=0, dtype="float32", device=dev)
    sd = spectral.sparsify(dec, int(round(a.density * cfg.n * cfg.r)))
    del dec
    torch.cuda.empty_cache()
    queries = ranking.QueryBatch(cfg.n, y_ptr, y_idx, y_val)
    h = ranking.h_alpha(0.99)
    flush = bench.L2Flush(dev)
    ctx.enable_timing(True)
    out = {"density": a.density, "nnz": sd.U_device.nnz, "rows": []}
    for b in [int(x) for x in a.batches.split(",")]:
        e = int(queries.y_ptr[b])
        qb = ranking.QueryBatch(cfg.n, queries.y_ptr[:b + 1], queries.y_idx[:e], queries.y_val[:e])
        dq = ranking.DeviceQueries(qb, sd.dtype, dev)
        res = ranking.FilterResult()
        for _ in range(3):
            ranking.filter_device(sd, h, dq, topk=100, want_x=False, out=res)
        torch.cuda.synchronize()
        ctx.stage_reset()
        ms = 0.0
        for _ in range(a.steps):
            flush()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ranking.filter_device(sd, h, dq, topk=100, want_x=False, out=res)
            e1.record()
            torch.cuda.synchronize()
            ms += e0.elapsed_time(e1)
        stages = {k: ctx.stage_time(k)[0] / a.steps for k in ("project", "filter_spmm", "topk")}
        fg = ranking.FilterGraph(sd, h, b=b, nnz_cap=int(qb.y_ptr[-1]), topk=100)
        fg.stage(qb)
        for _ in range(3):
            fg.replay()
        torch.cuda.synchronize()
        gms = 0.0
        for _ in range(a.steps):
            flush()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fg.replay()
            e1.record()
            torch.cuda.synchronize()
            gms += e0.elapsed_time(e1)
        if b == 1:
            torch.cuda.nvtx.range_push("k9s:b1")
            for _ in range(5):
                flush()
                fg.replay()
            torch.cuda.synchronize()
            torch.cuda.nvtx.range_pop()
        row = {"b": b, "path": ctx.last_online_path, "eager_ms": ms / a.steps, "graph_ms": gms / a.steps,
               "graph_qps": b * a.steps / (gms / 1e3), "stage_ms": stages}
        out["rows"].append(row)
        print(json.dumps(row), flush=True)
        del fg, res, dq
    print(json.dumps(out))


if __name__ == "__main__":
    main()
