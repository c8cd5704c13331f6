"""CholeskyQR2 (spectral.orthonormalize) at C3 shape with per-stage device times.

    python tools/orth_micro.py [--n 1000000] [--k 5500] [--fast-apply 0|1]
"""

import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_1703_06935_b200 import _native as N  # noqa: E402
from paper_1703_06935_b200 import spectral  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--k", type=int, default=5500)
    ap.add_argument("--fast-apply", type=int, default=1)
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    spectral.FAST_FIRST_APPLY = bool(a.fast_apply)
    dev = torch.device("cuda", 0)
    ctx = N.Context.get(dev)
    g = torch.Generator(device=dev)
    g.manual_seed(0)
    Y0 = torch.randn(a.n, a.k, generator=g, device=dev)
    Y0 *= torch.linspace(0.1, 1.0, a.k, device=dev)[None, :]  # uneven column scales, like SpMM outputs
    Y = Y0.clone()
    spectral.orthonormalize(Y, ctx)  # warm-up (allocations, tensor maps)
    torch.cuda.synchronize()
    out = {"n": a.n, "k": a.k, "fast_apply": a.fast_apply}
    walls = []
    ctx.enable_timing(True)
    ctx.stage_reset()
    for _ in range(a.reps):
        Y.copy_(Y0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        stats = []
        spectral.orthonormalize(Y, ctx, stats)
        torch.cuda.synchronize()
        walls.append(time.perf_counter() - t0)
    out["wall_ms"] = [w * 1e3 for w in walls]
    out["stage_ms_per_call"] = {s: ctx.stage_time(s)[0] / a.reps for s in ("gram", "cholesky", "apply", "householder")}
    out["method"] = stats
    Qd = Y[:20000].double()
    out["orth_head"] = float((Qd.T @ Qd - torch.eye(a.k, device=dev, dtype=torch.float64)).abs().max())
    print(json.dumps(out))


if __name__ == "__main__":
    main()
