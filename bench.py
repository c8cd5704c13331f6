#!/usr/bin/env python
"""FSR hot-path benchmark on B200 (one JSON line on rank 0).

Headline (BASELINE.json metric "... online ranked queries/sec at n=1M"):
ranked queries per second of the online path -- K8 projection, K9 sparse
filtering, copy-uncovered, exact top-100 -- on the sparsified decomposition
of config C3 (n=1e6, r=5000, U~ density 2%), one step = one batch of b
k=50-sparse queries.  The offline part of the metric (simultaneous-iteration
time and SpMM HBM GB/s) is measured in the same run and reported under
"offline".

    python bench.py [--gpus N --steps K --warmup W] [--config C2|C3] [--impl reference]

Under torchrun each rank builds the same inputs, runs the offline pipeline as
a replica and answers its own query batches (weak scaling: b queries per GPU
per step); `value` = all ranks' queries / max-over-ranks device time.

`--impl reference` times the reference's CPU path -- the stock
``specrank.ranking.filter`` + ``rank`` installed into baseline/_ref (the
oracle port only when that is absent) -- on a structure-equivalent synthetic
decomposition (same n, r, tau) on host cores.  The offline half of the
metric gets a CPU baseline too (``offline.cpu_baseline``): the reference's
own numpy/scipy calls timed on samples and extrapolated at C3, and the full
stock ``decompose`` + ``sparsify`` at C1/C2.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

# BASELINE.json "metric", verbatim; `value` is its online ranked queries/s part,
# the offline SI time and SpMM GB/s are reported under "offline".
METRIC = "offline SI time & SpMM HBM GB/s; online ranked queries/sec at n=1M, 1\u20138 GPU"


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="fsr", choices=["fsr", "reference"])
    ap.add_argument("--config", default="C3", choices=["C1", "C2", "C3"])
    ap.add_argument("--n", type=int, default=None, help="override n (development)")
    ap.add_argument("--batch", type=int, default=1024)
    ap.add_argument("--density", type=float, default=None)
    ap.add_argument("--topk", type=int, default=100)
    ap.add_argument("--dtype", default="float32", choices=["float32", "float64"])
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--no-sweep", action="store_true", help="skip the C5 online sweep")
    ap.add_argument("--sweep-settle-s", type=float, default=0.5,
                    help="idle time before each small-batch (b <= 64) sweep point, so a latency point is not "
                         "measured at the clocks the power cap left behind after the wide-batch points")
    ap.add_argument("--no-parity", action="store_true", help="skip the full-size parity checks")
    ap.add_argument("--no-offline-warmup", action="store_true",
                    help="time the offline decomposition on its first (cold) run")
    ap.add_argument("--cpu-procs", type=int, default=64, help="processes for the CPU oracle arms (capped at nproc)")
    ap.add_argument("--offline-cpu-full", dest="offline_cpu_full", action="store_true", default=None,
                    help="also time the full stock reference decompose + sparsify (default at C1/C2)")
    ap.add_argument("--no-offline-cpu-full", dest="offline_cpu_full", action="store_false")
    return ap.parse_args()


def load_peaks():
    path = os.path.join(REPO, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def load_tensor_peak():
    """Dense fp16/bf16 tensor peak in TF/s: MEASURED_PEAKS.json's cuBLAS bf16
    (burst; kind::f16 and kind::bf16 run at the same rate), else the
    profiling recipe's fallback."""
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["bf16_tflops"]), "measured (cuBLAS bf16 burst)"
    except Exception:
        return 1600.0, "fallback"


def load_profile(name, rnd=None):
    """A committed measurement summary under profiles/ (None when absent)."""
    path = os.path.join(REPO, "profiles", rnd or PROFILE_ROUND, name)
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return None


PROFILE_ROUND = "r02"
FP32_LANES_PER_SM = 128  # FFMA lanes per SM (sm_100)


class ClockSampler:
    """nvidia-smi sampling of SM clocks and throttle reasons while the bench runs."""

    FIELDS = ["clocks.sm", "clocks.max.sm", "power.draw", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.lines = []
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(index), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < len(self.FIELDS):
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for name, flag in zip(self.NAMES, parts[3:]):
                if flag.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return None
        loaded = [s for s in sm if mx and s >= 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_min_mhz": min(loaded), "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# reference arm: the CPU oracle port of the reference's online path
# ---------------------------------------------------------------------------

def synthetic_sparse_decomposition(n, r, tau, seed=7):
    import scipy.sparse as sp

    rng = np.random.default_rng(seed)
    per = max(1, tau // n)
    cols = rng.integers(0, r, size=(n, per)).astype(np.int32)
    cols.sort(axis=1)
    vals = rng.standard_normal((n, per)) / math.sqrt(per)
    indptr = np.arange(0, n * per + 1, per, dtype=np.int64)
    U = sp.csr_matrix((vals.ravel(), cols.ravel(), indptr), shape=(n, r))
    U.sum_duplicates()
    lam = np.sort(rng.uniform(-0.2, 1.0, r))[::-1].copy()
    eta = np.sqrt(np.asarray(U.multiply(U).sum(axis=1)).ravel())
    return U, lam, eta


def synthetic_queries(n, b, k, seed=11):
    rng = np.random.default_rng(seed)
    ys = []
    for _ in range(b):
        idx = np.unique(rng.integers(0, n, size=k))
        ys.append((idx.astype(np.int64), rng.random(idx.size) ** 3))
    return ys


def load_reference():
    """The stock reference package ``specrank`` installed into baseline/_ref
    (``pip install --no-index --no-deps --target baseline/_ref`` of
    /root/reference/pkg; pure Python, so it travels to the GPU box with the
    repo snapshot).  None when it is absent."""
    ref = os.path.join(REPO, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "specrank")):
        return None
    if ref not in sys.path:
        sys.path.insert(0, ref)
    try:
        from specrank import graph as rgraph  # noqa: F401
        from specrank import ranking as rranking
        from specrank import spectral as rspectral
    except Exception:
        return None
    return {"ranking": rranking, "spectral": rspectral, "graph": rgraph, "path": ref}


def reference_decomposition(ref, U, lam, eta, r, tau):
    """Wrap a host CSR U~ (float64) as the reference's own SparseDecomposition."""
    S, G = ref["spectral"], ref["graph"]
    return S.SpectralDecomposition(U=U, eigenvalues=np.asarray(lam, dtype=np.float64),
                                   eta=np.asarray(eta, dtype=np.float64),
                                   components=G.ComponentLabeling.trivial(U.shape[0]), variant=S.Variant.SPARSE,
                                   provenance=S.Provenance(r=r, tau=tau, seed=0))


def time_oracle_queries(U, lam, eta, ys, alpha, budget_s, topk, ref=None):
    """Reference per-query path: filter (ranking.py:229-255) + rank[:topk]
    (ranking.py:390-395) -- the stock ``specrank`` functions when ``ref`` is
    given (U, lam, eta then describe a reference SpectralDecomposition),
    else the oracle port of the same lines."""
    if ref is not None:
        R = ref["ranking"]
        dec = reference_decomposition(ref, U, lam, eta, U.shape[1], U.nnz)
        h = R.h_alpha(alpha)
        n = U.shape[0]
        done, t0 = 0, time.perf_counter()
        while done < len(ys):
            idx, val = ys[done % len(ys)]
            y = R.ObservationVector(n, idx, val, cap=max(1, idx.size))
            x = R.filter(dec, h, y)
            R.rank(x)[:topk]
            done += 1
            if time.perf_counter() - t0 > budget_s and done >= 2:
                break
        return done, time.perf_counter() - t0
    from oracle import fsr_oracle as O

    w = O.transfer_values(O.h_alpha(alpha), lam)
    done, t0 = 0, time.perf_counter()
    while done < len(ys):
        idx, val = ys[done % len(ys)]
        x = O.filter_scores(U, lam, eta, w, idx, val)
        O.rank(x)[:topk]
        done += 1
        if time.perf_counter() - t0 > budget_s and done >= 2:
            break
    return done, time.perf_counter() - t0


_POOL_STATE = {}


def _oracle_worker(args):
    """One process of the parallel CPU arm: queries [lo, hi) of the shared list, within a budget."""
    lo, hi, budget_s, topk = args
    st = _POOL_STATE
    done, secs = time_oracle_queries(st["U"], st["lam"], st["eta"], st["ys"][lo:hi], st["alpha"], budget_s, topk,
                                     st.get("ref"))
    return done, secs


def parallel_oracle_qps(U, lam, eta, ys, alpha, budget_s, topk, procs, ref=None):
    """Queries/s of the reference's per-query path over `procs` forked
    processes (U shared copy-on-write).

    The reference's filter is single-threaded scipy (csr_matvec), so the CPU's
    best throughput comes from answering independent queries in parallel.
    Returns (queries done, wall seconds, processes used)."""
    import multiprocessing as mp

    if procs <= 1:
        done, secs = time_oracle_queries(U, lam, eta, ys, alpha, budget_s, topk, ref)
        return done, secs, 1
    _POOL_STATE.update(U=U, lam=lam, eta=eta, ys=ys, alpha=alpha, ref=ref)
    per = max(1, len(ys) // procs)
    chunks = [(i * per, (i + 1) * per if i < procs - 1 else len(ys), budget_s, topk) for i in range(procs)]
    chunks = [c for c in chunks if c[1] > c[0]]
    ctxm = mp.get_context("fork")
    t0 = time.perf_counter()
    with ctxm.Pool(len(chunks)) as pool:
        res = pool.map(_oracle_worker, chunks)
    wall = time.perf_counter() - t0
    _POOL_STATE.clear()
    return sum(d for d, _ in res), wall, len(chunks)


def cpu_kind(ref):
    return ("reference (stock specrank.ranking.filter + rank from baseline/_ref)" if ref is not None
            else "port (oracle/fsr_oracle.py restatement; baseline/_ref absent)")


def run_reference(args, cfg, n, rank, world):
    if rank != 0:
        return
    r = cfg.r
    density = args.density if args.density is not None else cfg.density
    tau = int(round(density * n * r))
    U, lam, eta = synthetic_sparse_decomposition(n, r, tau)
    ref = load_reference()
    procs = max(1, min(os.cpu_count() or 1, args.cpu_procs))
    # one step = one query per process, all processes in parallel (the reference has no batch API)
    ys = synthetic_queries(n, max((args.steps + args.warmup) * procs, 4), cfg.y_top)
    time_oracle_queries(U, lam, eta, ys[:args.warmup], cfg.alpha, 1e9, args.topk, ref)  # warm-up, untimed
    done, secs, procs = parallel_oracle_qps(U, lam, eta, ys[args.warmup * procs:], cfg.alpha, 1e9, args.topk, procs,
                                            ref)
    qps = done / secs
    cores = procs
    kind = "reference" if ref is not None else "port"
    line = {
        "metric": METRIC, "value": qps, "unit": "queries/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * secs / max(args.steps, 1), "queries": done,
        "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
        "config": {"workload": f"{cfg.name}/C5 online: {cpu_kind(ref)} on a synthetic U~ with n={n}, r={r}, "
                               f"tau={tau} (density {density}), k={cfg.y_top}-sparse y, h_alpha({cfg.alpha}), "
                               f"top-{args.topk}",
                   "step": f"one query per process on {cores} processes (reference has no batch API)"},
        "cpu_baseline": {"value": qps, "unit": "queries/s", "cores": cores, "kind": kind,
                         "sample": f"{done} queries, {secs:.1f} s wall, {cores} forked processes x scipy "
                                   f"csr_matvec (single-threaded each)" +
                                   (f"; specrank imported from {ref['path']}" if ref else "")},
        "e2e": {"value": qps, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def offline_cpu_baseline(S, n, r, r_hat, q, tau, panel_cols=256, panel_rows=16384, sort_rows=2048):
    """The reference's offline path timed per operation on this host's cores
    and extrapolated to the full config (the full CPU run is
    infeasible at C3 -- fp64 n x r_hat = 44 GB per array, QR hours).  Each
    timed call is the reference's own numpy/scipy call on a sample:
      SpMM  ``A.csr @ Q`` (spectral.py:170 -> sparsemat.py:63-64) on all n
            rows x ``panel_cols`` columns; scales with nnz * r_hat;
      QR    ``np.linalg.qr(block)`` (spectral.py:165) on ``panel_rows`` x r_hat;
            scales with the Householder count 4 m r_hat^2 - 4/3 r_hat^3
            (geqrf + orgqr);
      QtB   ``basis.Q.T @ basis.B`` (spectral.py:186) on panel_rows rows; linear in n;
      eigh  ``np.linalg.eigh(C)`` (spectral.py:188) on the full r_hat x r_hat: measured, no extrapolation;
      QV    ``basis.Q @ vecs`` (spectral.py:190) on panel_rows rows; linear in n;
      sparsify ``np.lexsort`` of the (-|u|, row, col) keys (spectral.py:281) on
            panel_rows x r entries; scales with N log N, N = n r.
    The orthogonality check after each QR (spectral.py:166-167, a Gram of Q)
    is counted as one more Q^T B-sized GEMM per round."""
    import scipy.sparse as sp

    ncpu = os.cpu_count() or 1
    t = {}
    A = sp.csr_matrix(S.csr, dtype=np.float64)
    rng = np.random.default_rng(0)
    Q = rng.standard_normal((n, panel_cols))
    t0 = time.perf_counter()
    A @ Q
    t["spmm_panel_s"] = time.perf_counter() - t0
    del Q
    m = min(panel_rows, n)
    P = rng.standard_normal((m, r_hat))
    t0 = time.perf_counter()
    np.linalg.qr(P)
    t["qr_panel_s"] = time.perf_counter() - t0
    P2 = rng.standard_normal((m, r_hat))
    t0 = time.perf_counter()
    P.T @ P2
    t["qtb_panel_s"] = time.perf_counter() - t0
    V = rng.standard_normal((r_hat, r))
    t0 = time.perf_counter()
    P @ V
    t["qv_panel_s"] = time.perf_counter() - t0
    del P2, V
    C = P.T @ P / m
    t0 = time.perf_counter()
    np.linalg.eigh(C)
    t["eigh_s"] = time.perf_counter() - t0
    del P, C
    ms = min(sort_rows, n)
    N_s = ms * r
    u = rng.standard_normal(N_s)
    rows = np.repeat(np.arange(ms), r)
    cols = np.tile(np.arange(r), ms)
    t0 = time.perf_counter()
    np.lexsort((cols, rows, -np.abs(u)))
    t["lexsort_panel_s"] = time.perf_counter() - t0
    del u, rows, cols

    def hh(rows_):
        return 4.0 * rows_ * r_hat ** 2 - 4.0 / 3.0 * r_hat ** 3

    spmm_s = t["spmm_panel_s"] * r_hat / panel_cols
    qr_s = t["qr_panel_s"] * hh(n) / hh(m)
    qtb_s = t["qtb_panel_s"] * n / m
    qv_s = t["qv_panel_s"] * n / m
    N = n * r
    sparsify_s = t["lexsort_panel_s"] * (N * math.log(N)) / (N_s * math.log(N_s))
    si_s = q * (qr_s + qtb_s + spmm_s)
    rr_s = qtb_s + t["eigh_s"] + qv_s
    spmm_bytes = A.nnz * 12 + (n + 1) * 4 + 2 * 8 * n * r_hat
    return {"kind": "extrapolated", "cores": ncpu,
            "threads": {"openblas": os.environ.get("OPENBLAS_NUM_THREADS", f"default ({ncpu})"),
                        "scipy_spmm": 1},
            "sample": f"reference calls on samples: A.csr @ Q[:, :{panel_cols}] (all {n} rows, nnz={A.nnz}); "
                      f"np.linalg.qr / Q^T B / Q V on {m} x {r_hat} row panels; eigh on the full {r_hat}^2; "
                      f"lexsort on {ms} x {r} entries",
            "measured_s": t,
            "si_time_s": si_s, "rayleigh_ritz_s": rr_s, "sparsify_s": sparsify_s,
            "decompose_total_s": si_s + rr_s + sparsify_s,
            "spmm_s_per_iter": spmm_s, "spmm_gbs": spmm_bytes / spmm_s / 1e9,
            "qr_s_per_iter": qr_s,
            "model": "SpMM x r_hat/panel_cols; QR x (4 n r_hat^2 - 4/3 r_hat^3)/(same at m rows); GEMMs x n/m; "
                     "sparsify x N log N; SI = q (QR + orthogonality Gram + SpMM)"}


def offline_cpu_full(S, r, p, q, tau):
    """The stock reference ``decompose`` + ``sparsify`` timed once in full
    (feasible at C2: n = 1e5).  Needs baseline/_ref."""
    import scipy.sparse as sp

    ref = load_reference()
    if ref is None:
        return None
    from specrank.sparsemat import SparseSymmetricMatrix as RefSSM

    A = RefSSM(sp.csr_matrix(S.csr, dtype=np.float64))
    t0 = time.perf_counter()
    dec = ref["spectral"].decompose(A, r, p=p, q=q, seed=0)
    t1 = time.perf_counter()
    ref["spectral"].sparsify(dec, tau)
    t2 = time.perf_counter()
    return {"kind": "reference", "cores": os.cpu_count() or 1, "decompose_s": t1 - t0, "sparsify_s": t2 - t1,
            "decompose_total_s": t2 - t0,
            "sample": "full stock specrank.spectral.decompose + sparsify on this config's W (fp64)"}


# ---------------------------------------------------------------------------
# FSR arm
# ---------------------------------------------------------------------------

KNN_STATS = {}  # rows of the last build_inputs settled by each certification stage (knn.certified_topk)


def build_inputs(cfg, n, n_queries, device, dtype):
    import torch

    from paper_1703_06935_b200 import graph, knn, workloads

    t0 = time.perf_counter()
    X, Qv, _ = workloads.device_cluster_descriptors(cfg, device, n=n, queries=n_queries)
    KNN_STATS.clear()
    # certified bf16 candidates, fp32 re-score
    W = knn.mutual_knn_graph_device(X, cfg.k, cfg.gamma, gemm_dtype=torch.bfloat16, stats=KNN_STATS)
    deg = graph.degrees_device(W, device)
    S = graph.normalize_adjacency(W, deg, dtype=dtype, device=device)
    y_ptr, y_idx, y_val = knn.observation_batch_device(Qv, X, cfg.y_top, cfg.gamma)
    del X, Qv
    torch.cuda.synchronize()
    return S, (y_ptr, y_idx, y_val), time.perf_counter() - t0, int(W.nnz), int((deg == 0).sum())


def sharded_offline(S, r, r_hat, q, tau, dt, device, ev):
    """Row-sharded SI + Rayleigh-Ritz + threshold over NCCL; U~ replicated afterwards."""
    import torch

    from paper_1703_06935_b200 import distributed as D
    from paper_1703_06935_b200 import spectral
    from paper_1703_06935_b200.graph import ComponentLabeling

    comm = D.Comm()
    ops = D.CudaOps(device, dt)
    A = S.device(ops.dt_t, device)
    shard = D.make_shard(comm, A.indptr.cpu().numpy())
    A_local = D.shard_rows(A, shard.r0, shard.r1)
    ev[0].record()
    Q, B = D.sharded_range_finder(comm, ops, A_local, shard, r_hat, q, 0, ops.dt)
    ev[1].record()
    U, lam, _ = D.sharded_rayleigh_ritz(comm, ops, Q, B, r, shard)
    del Q, B
    ev[2].record()
    Ut, eta_s, _ = D.sharded_sparsify(comm, ops, U, tau, shard, ops.dt)
    del U
    full = D.gather_csr(comm, Ut, shard)
    eta = comm.all_gather_rows(eta_s.unsqueeze(1), shard.counts).squeeze(1).contiguous()
    ev[3].record()
    return spectral.SpectralDecomposition(full, lam, eta, ComponentLabeling.trivial(shard.n),
                                          spectral.Variant.SPARSE, spectral.Provenance(r=r, p=r_hat - r, q=q,
                                                                                       tau=tau, seed=0))


def offline_properties(S, dec, sdec, tau, device, ctx, m=64):
    """Size-independent checks of the full-size decomposition (untimed, N=1):
    Ritz identity lambda_i = u_i^T W u_i and u_i^T u_j = delta_ij on m sampled
    columns, and the sparsify contract (U~ keeps exactly tau entries, all
    at least as large in |u| as every dropped one)."""
    import torch

    from paper_1703_06935_b200 import _native as N
    from paper_1703_06935_b200 import spectral

    U = dec.U_device
    n, r = U.shape
    cols = torch.as_tensor(np.unique(np.linspace(0, r - 1, m).round().astype(np.int64)), device=device)
    Us = U.index_select(1, cols).contiguous()
    Bs = torch.empty_like(Us)
    Ad = S.device(Us.dtype, device)
    spectral._spmm(ctx, N.dtype_code(Us.dtype), Ad, Us, Bs)
    U64, B64 = Us.double(), Bs.double()
    rho = (U64 * B64).sum(0).cpu().numpy()
    lam = dec.eigenvalues[cols.cpu().numpy()]
    G = (U64.T @ U64).cpu().numpy()
    res = torch.linalg.vector_norm(B64 - U64 * torch.as_tensor(lam, device=device), dim=0).cpu().numpy()
    del Us, Bs, U64, B64
    kept = sdec.U_device.values.abs()
    t = float(kept.min())
    gt = ge = 0
    for i0 in range(0, n, 65536):
        blk = U[i0:i0 + 65536].abs()
        gt += int((blk > t).sum())
        ge += int((blk >= t).sum())
    scale = float(np.max(np.abs(dec.eigenvalues)))
    return {"sample_columns": int(cols.numel()),
            "ritz_identity_max_rel": float(np.max(np.abs(rho - lam)) / scale), "ritz_tol": 1e-5,
            "orthonormality_max_abs": float(np.max(np.abs(G - np.eye(G.shape[0])))),
            "residual_norm_top1": float(res[0]), "residual_norm_median": float(np.median(res)),
            "sparsify_kept": int(sdec.U_device.nnz), "tau": int(tau),
            "sparsify_count_above_min_kept": gt, "sparsify_count_at_least_min_kept": ge,
            "sparsify_support_is_top_tau": bool(gt <= tau <= ge) and int(sdec.U_device.nnz) == int(tau)}


def online_parity(sdec, Uh, eta, queries, alpha, K, device, nq=8):
    """GPU scores / top-K vs the oracle port (scipy CSR f64) on the same
    GPU-produced U~ for nq full-size queries (north_star: x <= 1e-4 rel-L2,
    top-100 overlap >= 99%)."""
    from oracle import fsr_oracle as O
    from paper_1703_06935_b200 import ranking

    nq = min(nq, queries.b)
    e = int(queries.y_ptr[nq])
    qb = ranking.QueryBatch(queries.size, queries.y_ptr[:nq + 1], queries.y_idx[:e], queries.y_val[:e])
    h = ranking.h_alpha(alpha)
    dq = ranking.DeviceQueries(qb, sdec.dtype, device)
    res = ranking.filter_device(sdec, h, dq, topk=K, want_x=True)
    X = res.X.double().cpu().numpy()
    top = res.top_idx.cpu().numpy()
    w = O.transfer_values(O.h_alpha(alpha), sdec.eigenvalues)
    errs, overlaps, same = [], [], 0
    for j in range(nq):
        idx = qb.y_idx[qb.y_ptr[j]:qb.y_ptr[j + 1]]
        val = qb.y_val[qb.y_ptr[j]:qb.y_ptr[j + 1]]
        x = O.filter_scores(Uh, sdec.eigenvalues, eta, w, idx, val)
        errs.append(float(np.linalg.norm(X[j] - x) / np.linalg.norm(x)))
        ref_top = O.rank(x)[:K]
        overlaps.append(len(np.intersect1d(ref_top, top[j])) / K)
        same += int(np.array_equal(ref_top, top[j]))
    return {"queries": nq, "x_rel_l2_max": max(errs), "x_tol": 1e-4, "topk_overlap_min": min(overlaps),
            "topk_identical_order": same, "oracle": "oracle/fsr_oracle.py filter_scores + rank (scipy CSR f64)"}


def online_sweep(dec, sdec_default, density_default, cfg, n, r, queries, device, ctx, es, steps=3, warmup=2,
                 settle_s=0.0):
    """BASELINE C5: batches {1, 64, 1024, 10000} x U~ density {1, 2, 5}% with h_alpha(0.99),
    plus h_alpha(0.9) and heat exp(-10(1-x)) at 2% / b=1024.  Device-resident, top-100."""
    import torch

    from paper_1703_06935_b200 import ranking, spectral

    out = []
    flush = L2Flush(device)
    dens = sorted({0.01, 0.02, 0.05, density_default})
    batches = [1, 64, 1024, 10000]
    pool = queries.b
    for d in dens:
        sd = sdec_default if d == density_default else spectral.sparsify(dec, int(round(d * n * r)))
        tfs = [("h_alpha(0.99)", ranking.h_alpha(0.99))]
        if d == 0.02:
            tfs += [("h_alpha(0.9)", ranking.h_alpha(0.9)), ("heat(10)", ranking.heat_kernel(10.0))]
        for b in batches:
            if b > pool:
                reps = -(-b // pool)
                qb = ranking.QueryBatch(n, *_repeat_batch(queries, reps, b))
            else:
                e = queries.y_ptr[b]
                qb = ranking.QueryBatch(n, queries.y_ptr[:b + 1], queries.y_idx[:e], queries.y_val[:e])
            dq = ranking.DeviceQueries(qb, sd.dtype, device)
            for name, h in tfs:
                if name != "h_alpha(0.99)" and b != 1024:
                    continue
                res = ranking.FilterResult()
                if b <= 64 and settle_s > 0:
                    torch.cuda.synchronize()
                    time.sleep(settle_s)
                for _ in range(warmup if b > 64 else max(warmup, 5)):
                    ranking.filter_device(sd, h, dq, topk=100, want_x=False, out=res)
                torch.cuda.synchronize()
                ctx.stage_reset()
                ms = 0.0
                nsteps = 20 if b <= 64 else steps  # small batches: more samples (sub-millisecond steps)
                for _ in range(nsteps):
                    flush()
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    ranking.filter_device(sd, h, dq, topk=100, want_x=False, out=res)
                    e1.record()
                    torch.cuda.synchronize()
                    ms += e0.elapsed_time(e1)
                k9_ms, k9_cnt = ctx.stage_time("filter_spmm")
                kept = sd.U_device.nnz
                pth = ctx.last_online_path
                k9_bytes = kept * (es + 4) + (n + 1) * 8 + (2 if pth == "pruned" else es) * r * b + es * n * b
                row = {"density": d, "b": b, "h": name, "k9_path": pth,
                       "queries_per_s": b * nsteps / (ms / 1e3),
                       "ms_per_batch": ms / nsteps, "k9_ms": k9_ms / max(k9_cnt, 1)}
                if pth == "tc":
                    row["k9t_dense_tflops"] = 2.0 * n * r * b / (k9_ms / max(k9_cnt, 1) * 1e-3) / 1e12
                elif pth == "stream":
                    # K9s select pass: per group of <= 8 queries the packed U~ (4 B per entry),
                    # indptr (8 B) and the bound factors (4 B) per row stream from HBM once
                    nb = next(v for v in (8, 4, 2, 1) if v <= b)
                    s_bytes = -(-b // nb) * (4 * kept + 12 * n)
                    row["k9s_stream_gbs"] = s_bytes / (k9_ms / max(k9_cnt, 1) * 1e-3) / 1e9
                    row["k9s_hbm_frac"] = row["k9s_stream_gbs"] / load_peaks()[0]
                elif pth == "sell":
                    # K9e: per pass of 1 / 2 / 4 queries the sliced-ELL entries (6 B each) and the row
                    # metadata (perm, lens: 8 B per row) stream from HBM once; x is scattered (4 B per row and query)
                    nbq = 1 if b == 1 else (2 if b == 2 else 4)
                    lay = ranking.sell_layout(sd)
                    s_bytes = -(-b // nbq) * (6 * int(lay[3].numel()) + 8 * n) + 4 * n * b
                    row["k9e_stream_gbs"] = s_bytes / (k9_ms / max(k9_cnt, 1) * 1e-3) / 1e9
                    row["k9e_hbm_frac"] = row["k9e_stream_gbs"] / load_peaks()[0]
                else:
                    row["k9_algorithmic_gbs"] = k9_bytes / (k9_ms / max(k9_cnt, 1) * 1e-3) / 1e9
                row["useful_fp32_tflops"] = 2.0 * kept * b / (k9_ms / max(k9_cnt, 1) * 1e-3) / 1e12
                if b <= 64 and name == "h_alpha(0.99)":
                    row.update(graph_sweep_row(sd, h, qb, b, nsteps, max(warmup, 5), flush, ctx))
                    row["settle_s"] = settle_s
                out.append(row)
                del res
            del dq
        if sd is not sdec_default:
            del sd
        torch.cuda.empty_cache()
    return out


def graph_sweep_row(sd, h, qb, b, steps, warmup, flush, ctx):
    """Same step through ranking.FilterGraph (one CUDA-graph launch per batch):
    device time per replay, and host-to-host latency (stage + replay + top-k D2H)."""
    import torch

    from paper_1703_06935_b200 import ranking

    timing = ctx._timing
    fg = ranking.FilterGraph(sd, h, b=b, nnz_cap=int(qb.y_ptr[-1]), topk=100)
    fg.stage(qb)
    for _ in range(warmup):
        fg.replay()
    torch.cuda.synchronize()
    ms = 0.0
    for _ in range(steps):
        flush()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fg.replay()
        e1.record()
        torch.cuda.synchronize()
        ms += e0.elapsed_time(e1)
    lat = []
    for _ in range(steps):
        flush()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        res = fg.run(qb)
        res.top_idx.cpu()
        res.top_val.cpu()
        lat.append(time.perf_counter() - t0)
    ctx.enable_timing(timing)
    del fg
    return {"graph_ms_per_batch": ms / steps, "graph_queries_per_s": b * steps / (ms / 1e3),
            "graph_e2e_latency_ms": 1e3 * min(lat)}


def _repeat_batch(queries, reps, b):
    ptr = [0]
    idx, val = [], []
    for j in range(b):
        k = j % queries.b
        s, e = queries.y_ptr[k], queries.y_ptr[k + 1]
        idx.append(queries.y_idx[s:e])
        val.append(queries.y_val[s:e])
        ptr.append(ptr[-1] + (e - s))
    return np.asarray(ptr, np.int64), np.concatenate(idx), np.concatenate(val)


class L2Flush:
    """Untimed L2 flush between timed steps: write a 256 MB buffer (> 126 MB L2),
    then read a second one so the dirty lines are written back before the
    timed region starts (otherwise their write-back lands inside it)."""

    def __init__(self, device):
        import torch

        self.w = torch.empty(256 << 20, dtype=torch.uint8, device=device)
        self.r = torch.zeros(64 << 20, dtype=torch.float32, device=device)

    def __call__(self):
        self.w.zero_()
        self.r.sum()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    dev = "cpu" if dist.get_backend() == "gloo" else "cuda"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def run_fsr(args, cfg, n, rank, world, local_rank):
    import torch

    from paper_1703_06935_b200 import _native as N
    from paper_1703_06935_b200 import ranking, spectral

    device = torch.device("cuda", local_rank)
    torch.cuda.set_device(device)
    peak_gbs, peak_kind = load_peaks()
    dt = args.dtype
    es = 4 if dt == "float32" else 8
    density = args.density if args.density is not None else cfg.density
    r, r_hat, q = cfg.r, min(cfg.r + cfg.p, n), cfg.q
    tau = int(round(density * n * r))
    b = args.batch
    n_batches = 4
    n_queries = b * n_batches * world

    S, (y_ptr, y_idx, y_val), t_inputs, nnz_w, isolated = build_inputs(cfg, n, n_queries, device, dt)
    all_queries = ranking.QueryBatch(n, y_ptr, y_idx, y_val)
    ctx = N.Context.get(device)

    # ---------------- offline: SI + Rayleigh-Ritz + sparsify ------------------
    # One untimed pass first: it sizes libfsr's scratch arena and torch's
    # allocator pools (multi-GB first-touch cudaMalloc/cudaFree inside the
    # dense stages made single-shot timings swing by up to 2x), then the timed pass.
    if not args.no_offline_warmup:
        if world == 1:
            _b = spectral.range_finder(S, r_hat, q, 0, dtype=dt, device=device,
                                       _orthonormal_last=not spectral.fused_rr_enabled(dt))
            _d = spectral.approx_eigendecomposition(S, _b, r)
            del _b
            _s = spectral.sparsify(_d, tau)
            del _d, _s
        else:
            _s = sharded_offline(S, r, r_hat, q, tau, dt, device,
                                 [torch.cuda.Event(enable_timing=True) for _ in range(4)])
            del _s
        torch.cuda.synchronize()
    ctx.enable_timing(True)
    ctx.stage_reset()
    off_clocks = ClockSampler(local_rank)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_push("fsr:offline")
    if world == 1:
        ev[0].record()
        # the same schedule as spectral.decompose (timed in two parts)
        basis = spectral.range_finder(S, r_hat, q, 0, dtype=dt, device=device,
                                      _orthonormal_last=not spectral.fused_rr_enabled(dt))
        ev[1].record()
        dec = spectral.approx_eigendecomposition(S, basis, r)
        del basis
        ev[2].record()
        sdec = spectral.sparsify(dec, tau)
        ev[3].record()
        if args.no_sweep:
            del dec
    else:
        sdec = sharded_offline(S, r, r_hat, q, tau, dt, device, ev)
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    off_clk = off_clocks.stop()
    stages = {name: ctx.stage_time(name) for name in N.STAGES}
    torch.cuda.empty_cache()
    si_s = max_over_ranks(ev[0].elapsed_time(ev[1]) / 1e3, world)
    rr_s = max_over_ranks(ev[1].elapsed_time(ev[2]) / 1e3, world)
    sp_s = max_over_ranks(ev[2].elapsed_time(ev[3]) / 1e3, world)
    spmm_ms, spmm_cnt = stages["spmm"]
    # per-iteration time of the slowest rank; the byte counts below are whole-matrix,
    # so the GB/s figures are job aggregates and the fractions are over world x peak
    spmm_ms_iter = max_over_ranks(spmm_ms / max(spmm_cnt, 1), world)
    nnz_s = S.nnz
    spmm_bytes = nnz_s * (es + 4) + (n + 1) * 8 + 2 * es * n * r_hat
    spmm_gbs = spmm_bytes / (spmm_ms_iter * 1e-3) / 1e9
    # what K2 must actually move on a graph without locality: one dense row
    # gather per nonzero (Q >> L2), i.e. nnz * r_hat * es bytes from DRAM
    spmm_gather = nnz_s * r_hat * es
    spmm_gather_gbs = spmm_gather / (spmm_ms_iter * 1e-3) / 1e9
    offline = {
        "si_time_s": si_s, "rayleigh_ritz_s": rr_s, "sparsify_s": sp_s, "decompose_total_s": si_s + rr_s + sp_s,
        "spmm_ms_per_iter": spmm_ms_iter, "spmm_launches": spmm_cnt, "spmm_algorithmic_bytes": spmm_bytes,
        "spmm_gbs": spmm_gbs, "spmm_hbm_frac": spmm_gbs / (world * peak_gbs),
        "spmm_gather_bytes": spmm_gather, "spmm_gather_gbs": spmm_gather_gbs,
        "spmm_gather_hbm_frac": spmm_gather_gbs / (world * peak_gbs),
        "spmm_fp32_tflops": 2.0 * nnz_s * r_hat / (spmm_ms_iter * 1e-3) / 1e12,
        "stage_ms": {k: round(v[0], 3) for k, v in stages.items() if v[1]},
        "nnz_W": nnz_w, "isolated_vertices": isolated, "kept_nnz": sdec.U_device.nnz, "inputs_build_s": t_inputs,
        "knn_certified_rows": dict(KNN_STATS),
        "clocks": off_clk,
        "timed_run": "second of two identical runs (the first sizes allocations)" if not args.no_offline_warmup
                     else "first run",
    }

    # ---------------- online: device-resident batches ------------------------
    h = ranking.h_alpha(cfg.alpha)
    per_rank = [all_queries.split(world * n_batches, rank * n_batches + i) for i in range(n_batches)]
    dqs = [ranking.DeviceQueries(qb, sdec.dtype, device) for qb in per_rank]
    K = args.topk
    res = ranking.FilterResult(top_idx=torch.empty(b, K, dtype=torch.int64, device=device),
                               top_val=torch.empty(b, K, dtype=sdec.dtype, device=device))
    ws = torch.empty(ranking.filter_workspace_bytes(sdec, b, want_x=False, topk=K), dtype=torch.uint8,
                     device=device)
    path = ranking.online_path(sdec, b, K, ctx)
    if path == "tc":
        ranking.dense_layout(sdec)  # built once per decomposition, outside the timed region
    flush = L2Flush(device)  # > L2 (126 MB)

    def step(i):
        ranking.filter_device(sdec, h, dqs[i % n_batches], topk=K, want_x=False, out=res, workspace=ws)

    clocks = ClockSampler(local_rank)
    for i in range(args.warmup):
        step(i)
    torch.cuda.synchronize()
    ctx.stage_reset()
    launches0 = ctx.launches
    barrier(world)
    torch.cuda.synchronize()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    torch.cuda.nvtx.range_push("fsr:online")
    for i in range(args.steps):
        flush()  # untimed: evict U~ / Zs from L2 between steps
        starts[i].record()
        step(i)
        ends[i].record()
    torch.cuda.synchronize()
    torch.cuda.nvtx.range_pop()
    barrier(world)
    launches = ctx.launches - launches0
    dev_ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    on_stages = {name: ctx.stage_time(name) for name in ("project", "filter_spmm", "copy_uncovered", "topk")}
    dev_ms_max = max_over_ranks(dev_ms, world)
    value = world * b * args.steps / (dev_ms_max / 1e3)

    # roofline of the dominant kernel: the main K9t GEMM (tensor), or K9 / K9h
    # (sparse U~ x Zs, HBM by the survey's count; K9h gathers Zs in fp16)
    k9_ms, k9_cnt = on_stages["filter_spmm"]
    k9_ms_launch = k9_ms / max(k9_cnt, 1)
    kept = sdec.U_device.nnz
    k9_share = k9_ms / max(sum(v[0] for v in on_stages.values()), 1e-9)
    certified = path in ("tc", "pruned")
    tc_stats = None
    if path == "tc":
        st2 = ranking.last_tc_stats(ws, sdec, b)
        tc_stats = {"candidates_median": float(np.median(st2[:, 0])), "candidates_max": int(st2[:, 0].max()),
                    "rescored_median": float(np.median(st2[:, 1])), "rescored_max": int(st2[:, 1].max())}
    # certified paths: same top-k as the unpruned fp32 path, bit for bit (untimed check)
    prune_check = None
    if certified:
        same, fallback = True, 0
        for dq in dqs:
            ranking.filter_device(sdec, h, dq, topk=K, want_x=False, out=res, workspace=ws)
            torch.cuda.synchronize()
            fallback += ranking.last_fallback_count(ws, sdec, b, ctx)
            pi, pv = res.top_idx.clone(), res.top_val.clone()
            ctx.set_topk_prune(False)
            ranking.filter_device(sdec, h, dq, topk=K, want_x=False, out=res, workspace=ws)
            torch.cuda.synchronize()
            ctx.set_topk_prune(True)
            same &= bool(torch.equal(pi, res.top_idx) and torch.equal(pv.view(torch.int32), res.top_val.view(torch.int32)))
        # the same timed protocol on the unpruned fp32 path, for reference
        ctx.set_topk_prune(False)
        for i in range(args.warmup):
            step(i)
        torch.cuda.synchronize()
        ums = 0.0
        for i in range(args.steps):
            flush()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            step(i)
            e1.record()
            torch.cuda.synchronize()
            ums += e0.elapsed_time(e1)
        ctx.set_topk_prune(True)
        ums = max_over_ranks(ums, world)
        prune_check = {"path": path, "batches": len(dqs), "topk_identical_to_unpruned_fp32": same,
                       "fallback_queries": fallback, "selection": tc_stats,
                       "unpruned_fp32": {"value": world * b * args.steps / (ums / 1e3), "unit": "queries/s",
                                         "ms_per_step": ums / args.steps}}
    profile_ok = cfg.name == "C3" and b == 1024 and es == 4 and args.density is None
    if path == "tc":
        tpeak, tpeak_kind = load_tensor_peak()
        ldr = (r + 7) // 8 * 8
        dense_flops = 2.0 * n * r * b
        achieved = dense_flops / (k9_ms_launch * 1e-3) / 1e12
        hbm_bytes = n * ldr * 2 + b * ldr * 2 + n * 4  # dense fp16 U~ once, fp16 Zh, c_i
        ncu9 = load_profile("k9t_ncu_full.json") or {}
        roofline = {
            "kernel": "K9t main pass k9t_gemm2sm_kernel<1> (tcgen05.mma.cta_group::2 kind::f16 M=256 N=256 on CTA "
                      "pairs, 4-CTA clusters with the U~ tile multicast across the pairs, 6 TMA stages, "
                      "double-buffered TMEM accumulators, fused certified selection)",
            "bound": "tensor", "achieved": achieved, "peak": tpeak, "unit": "TFLOP/s", "frac": achieved / tpeak,
            "peak_kind": tpeak_kind,
            "traffic": ncu9.get("dram_bytes_per_launch") if profile_ok else None,
            "traffic_source": "profiles/%s/k9t_ncu_full.json" % PROFILE_ROUND if (profile_ok and ncu9) else None,
            "algorithmic_flops_per_launch": dense_flops,
            "algorithmic_bytes_per_launch": hbm_bytes,
            "ms_per_launch": k9_ms_launch, "share_of_step": k9_share,
            "binding_limbs": {
                "hbm": {"bytes_per_launch": hbm_bytes, "achieved_gbs": hbm_bytes / (k9_ms_launch * 1e-3) / 1e9,
                        "peak_gbs": peak_gbs,
                        "frac": hbm_bytes / (k9_ms_launch * 1e-3) / 1e9 / peak_gbs},
                "useful_flops": {"flops_per_launch": 2.0 * kept * b,
                                 "achieved_tflops": 2.0 * kept * b / (k9_ms_launch * 1e-3) / 1e12,
                                 "note": "2 tau b: the products with a nonzero of U~ (the dense GEMM multiplies "
                                         "the zeros too: n r / tau = %.0fx the work, at tensor-core rate)"
                                         % (n * r / kept)},
            }}
    else:
        zb_es = 2 if path == "pruned" else es
        k9_bytes = kept * (es + 4) + (n + 1) * 8 + zb_es * r * b + es * n * b
        k9_gbs = k9_bytes / (k9_ms_launch * 1e-3) / 1e9
        k9_gather = kept * b * zb_es  # every nonzero of U~ gathers one b-wide row of Zs (L2-resident)
        k9_gather_gbs = k9_gather / (k9_ms_launch * 1e-3) / 1e9
        l2 = load_profile("l2_bw.json", "r01") or {}
        l2_peak = l2.get("gather_1KB_rows_19MB_GBs")
        ncu9 = load_profile("k9h_ncu_full.json" if path == "pruned" else "k9_ncu_full.json", "r01") or {}
        sms_ = torch.cuda.get_device_properties(device).multi_processor_count
        fp32_peak_ = 2.0 * sms_ * FP32_LANES_PER_SM * 1965.0 * 1e6 / 1e12
        roofline = {
            "kernel": ("K9h filter SpMM (spmm_T_half_kernel on U~ x fp16 Zs)" if path == "pruned" else
                       "K9 filter SpMM (spmm_rowpanel_T_kernel on U~ x Zs)"), "bound": "hbm",
            "achieved": k9_gbs, "peak": peak_gbs, "unit": "GB/s", "frac": k9_gbs / peak_gbs,
            "peak_kind": peak_kind, "traffic": ncu9.get("dram_bytes_per_launch") if profile_ok else None,
            "traffic_source": "profiles/r01/%s" % ("k9h_ncu_full.json" if path == "pruned" else "k9_ncu_full.json"),
            "algorithmic_bytes_per_launch": k9_bytes, "ms_per_launch": k9_ms_launch, "share_of_step": k9_share,
            "binding_limbs": {
                "l2_gather": {"bytes_per_launch": k9_gather, "achieved_gbs": k9_gather_gbs, "peak_gbs": l2_peak,
                              "frac": (k9_gather_gbs / l2_peak) if l2_peak else None,
                              "peak_source": "tools/l2_bw.cu random 1 KB row gathers (profiles/r01/l2_bw.json)"},
                "fp32_fma": {"achieved_tflops": 2.0 * kept * b / (k9_ms_launch * 1e-3) / 1e12,
                             "peak_tflops": fp32_peak_,
                             "frac": 2.0 * kept * b / (k9_ms_launch * 1e-3) / 1e12 / fp32_peak_}}}

    # ---------------- e2e through the public API with host buffers ----------
    # ranking.FilterGraph: host batch -> pinned staging -> one CUDA-graph launch
    # (H2D copies + K8 + K9 + copy-uncovered + top-k) -> top-k D2H into pinned
    # host memory; two graphs alternate so batch i+1 is staged while batch i runs
    e2e = None
    if not args.skip_e2e:
        host_batches = per_rank
        cap = max(int(qb.y_ptr[-1]) for qb in host_batches)
        fgs = [ranking.FilterGraph(sdec, h, b=b, nnz_cap=cap, topk=K) for _ in range(2)]
        for i in range(args.warmup):
            fgs[i % 2].submit(host_batches[i % n_batches])
            fgs[i % 2].fetch()
        torch.cuda.synchronize()
        barrier(world)
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record()
        d2h = 0
        for i in range(args.steps):
            fgs[i % 2].submit(host_batches[i % n_batches])
            if i >= 1:
                ti, tv = fgs[(i - 1) % 2].fetch()
                d2h += ti.nbytes + tv.nbytes
        ti, tv = fgs[(args.steps - 1) % 2].fetch()
        d2h += ti.nbytes + tv.nbytes
        t1.record()
        torch.cuda.synchronize()
        e2e_ms = max_over_ranks(t0.elapsed_time(t1), world)
        fg = fgs[0]
        h2d = fg.h_all.numel()  # one copy of the (y_ptr | y_idx | y_val) staging buffer per step
        e2e = {"value": world * b * args.steps / (e2e_ms / 1e3), "unit": "queries/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h // args.steps,
               "api": "ranking.FilterGraph.submit/fetch x2 (pinned staging + one CUDA-graph launch: H2D, K8, K9, "
                      "top-k; async top-k D2H)"}
        del fgs
    clk = clocks.stop()

    # ---------------- full-size parity (untimed, N=1) -------------------------
    parity = None
    if world == 1 and not args.no_parity:
        parity = {"offline": offline_properties(S, dec, sdec, tau, device, ctx) if not args.no_sweep else None}

    # ---------------- C5 online sweep (BASELINE config 5) ----------------------
    sweep = None
    if world == 1 and not args.no_sweep:
        del ws, res
        sweep = online_sweep(dec, sdec, density, cfg, n, r, all_queries, device, ctx, es,
                             settle_s=args.sweep_settle_s)
        del dec

    # ---------------- CPU baseline (rank 0, N=1) -----------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        Uh = sdec.U_device.to_scipy()
        eta = sdec.eta
        procs = max(1, min(os.cpu_count() or 1, args.cpu_procs))
        ys = [(all_queries.y_idx[all_queries.y_ptr[j]:all_queries.y_ptr[j + 1]],
               all_queries.y_val[all_queries.y_ptr[j]:all_queries.y_ptr[j + 1]])
              for j in range(min(all_queries.b, 8 * procs))]
        ref = load_reference()
        done, secs, procs = parallel_oracle_qps(Uh, sdec.eigenvalues, eta, ys, cfg.alpha, args.cpu_seconds, K,
                                                procs, ref)
        if parity is not None:
            parity["online"] = online_parity(sdec, Uh, eta, all_queries, cfg.alpha, K, device)
        cpu = {"value": done / secs, "unit": "queries/s", "cores": procs, "kind": "reference" if ref else "port",
               "sample": f"{done} queries of this workload on the GPU-produced U~ (scipy CSR f64), "
                         f"{cpu_kind(ref)}, {procs} forked processes, {secs:.1f} s wall"}

    # offline half of the metric: the reference's offline path on this host,
    # per operation and extrapolated (C3), or in full at C2 (rank 0, N=1)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            ocpu = offline_cpu_baseline(S, n, r, r_hat, q, tau)
            for k in ("si_time_s", "rayleigh_ritz_s", "sparsify_s", "decompose_total_s"):
                ocpu["speedup_" + k[:-2]] = ocpu[k] / max(offline[k], 1e-12)
            ocpu["speedup_spmm_per_iter"] = ocpu["spmm_s_per_iter"] / max(offline["spmm_ms_per_iter"] / 1e3, 1e-12)
            if args.offline_cpu_full or (args.offline_cpu_full is None and cfg.name in ("C1", "C2")):
                full = offline_cpu_full(S, r, r_hat - r, q, tau)
                if full is not None:
                    full["speedup_decompose_total"] = full["decompose_total_s"] / max(offline["decompose_total_s"],
                                                                                      1e-12)
                ocpu["full_run"] = full
        except Exception as exc:  # a host that cannot hold the samples must not lose the GPU line
            ocpu = {"error": f"{type(exc).__name__}: {exc}"}
        offline["cpu_baseline"] = ocpu

    if rank != 0:
        return
    sms = torch.cuda.get_device_properties(device).multi_processor_count
    fp32_peak = 2.0 * sms * FP32_LANES_PER_SM * ((clk or {}).get("sm_mhz") or 1965.0) * 1e6 / 1e12
    line = {
        "metric": METRIC, "value": value, "unit": "queries/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dev_ms_max / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32" if dt == "float32" else "f64",
        "data": "synthetic (seeded Gaussian clusters, BASELINE config shapes; datasets absent)",
        "config": {"workload": f"{cfg.name}/C5: n={n}, d={cfg.d}, k={cfg.k}, r={r}, p={cfg.p}, q={q}, "
                               f"U~ density {density} (tau={tau}), batch b={b} per GPU, y {cfg.y_top}-sparse, "
                               f"h_alpha({cfg.alpha}), top-{K}",
                   "global_batch": b * world, "parallelism": (f"offline row-sharded x{world} (NCCL all-gather + ordered fp64 sums), online replicas (batch split)" if world > 1 else "single GPU"),
                   "l2": "256 MB buffer written, then a 256 MB buffer read, between timed steps (L2 flush "
                         "with write-back outside the timed region); U~ itself > L2"},
        "online_path": {
            "tc": "K9t (csrc/k9t.cu): x~ = fp16 dense U~ x fp16 Zs on tcgen05 tensor cores (fp32 TMEM "
                  "accumulation), a rigorous per-row bound selects the rows that can reach the top-k inside the "
                  "GEMM epilogue (threshold from a 1/32 row-tile sample), those are re-scored exactly in fp32 in "
                  "the unpruned kernel's order -- the unpruned fp32 top-k bit for bit",
            "pruned": "certified pruned top-k: K9h gathers Zs rounded to fp16 (per-query power-of-two scale), "
                      "a rigorous per-row bound selects the rows that can reach the top-k, those are re-scored "
                      "exactly in fp32 in the unpruned kernel's order (csrc/prune.cuh)",
            "exact": "unpruned fp32 K9 + exact top-k"}[path],
        "prune_check": prune_check,
        "roofline": roofline,
        "online_stage_ms_per_step": {k: v[0] / args.steps for k, v in on_stages.items()},
        "offline": offline,
        "gpu_launches": launches,
        "e2e": e2e,
        "cpu_baseline": cpu,
        "clocks": clk,
        "c5_sweep": sweep,
        "parity": parity,
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    from paper_1703_06935_b200.workloads import CONFIGS

    cfg = CONFIGS[args.config]
    n = args.n or cfg.n
    if args.impl == "reference":
        run_reference(args, cfg, n, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        if os.environ.get("FSR_DIST_BACKEND") == "gloo":
            local_rank %= max(1, torch.cuda.device_count())  # functional check: ranks may share a GPU
        torch.cuda.set_device(local_rank)
        # FSR_DIST_BACKEND=gloo runs the multi-rank path with host-staged
        # collectives (e.g. two ranks sharing one GPU for a functional check)
        dist.init_process_group(os.environ.get("FSR_DIST_BACKEND", "nccl"))
    try:
        run_fsr(args, cfg, n, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
