"""Which orthonormalisation path each simultaneous-iteration round takes at C3
(fp32): spectral.range_finder's stats list, for the default and fused schedules."""

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
    S, _, _, _, _ = bench.build_inputs(cfg, cfg.n, 64, dev, "float32")
    r_hat = cfg.r + cfg.p
    from paper_1703_06935_b200 import _native as N

    ctx = N.Context.get(dev)
    out = {}
    for last in (True, False, True, False):
        st = []
        ctx.enable_timing(True)
        ctx.stage_reset()
        spectral.range_finder(S, r_hat, cfg.q, 0, dtype="float32", device=dev, stats=st, _orthonormal_last=last)
        times = {k: ctx.stage_time(k) for k in ("gram", "apply", "cholesky", "spmm", "gaussian")}
        ctx.enable_timing(False)
        out.setdefault("orthonormal_last" if last else "fused", []).append({"stats": st, "stages": times})
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
