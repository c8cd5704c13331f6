"""Time the parts of the certified bf16 kNN candidate step on one C3-sized block
(2048 query rows x n = 1e6 descriptors, d = 2048): the three bf16 GEMMs with
fp32 output, their sum, the top-(k+16) selection, the exact re-score."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1703_06935_b200 import knn, workloads  # noqa: E402
from paper_1703_06935_b200.workloads import CONFIGS  # noqa: E402


def main():
    cfg = CONFIGS["C3"]
    dev = torch.device("cuda", 0)
    X, _, _ = workloads.device_cluster_descriptors(cfg, dev, queries=16)
    hi = X.to(torch.bfloat16)
    lo = (X - hi.float()).to(torch.bfloat16)
    A = X[:2048]
    Ah, Al = hi[:2048], lo[:2048]
    out = {}

    def t(name, fn, reps=3):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            r = fn()
        torch.cuda.synchronize()
        out[name] = (time.perf_counter() - t0) / reps * 1e3
        return r

    mm = lambda a, b: torch.mm(a, b.T, out_dtype=torch.float32)  # noqa: E731
    t("gemm_bf16_ms", lambda: mm(Ah, hi))
    sims = t("gemm_bf16x3_ms", lambda: mm(Ah, hi) + mm(Ah, lo) + mm(Al, hi))
    cat = torch.cat([hi, lo, hi], dim=1)
    t("gemm_bf16x3_concatK_ms", lambda: mm(torch.cat([Ah, Ah, Al], dim=1), cat))
    top = t("topk66_ms", lambda: torch.topk(sims, 66, dim=1, sorted=False))
    t("topk66_libfsr_ms", lambda: knn._candidates_scored(sims, 66))
    t("rescore_ms", lambda: knn._rescore(A, X, top.indices))
    t("certified_topk_block_ms", lambda: knn.certified_topk(A, X, 50, 16, exclude_offset=0, split=(hi, lo, cat),
                                                           schemes=["bf16x3", "exact"]))
    out["blocks_at_C3"] = cfg.n / 2048
    print(json.dumps(out))


if __name__ == "__main__":
    main()
