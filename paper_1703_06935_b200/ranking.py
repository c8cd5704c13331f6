"""Online FSR ranking on the device: batched x = U h(Lambda) U^T y.

Drop-in for the reference ``ranking`` filtering entry points
(``ranking.py:23-155,219-255,390-395``): ``TransferFunction``, ``h_alpha``,
``custom_transfer``, ``ObservationVector``, ``filter`` and ``rank`` keep the
reference names, argument meaning and error behaviour.  ``filter_batch``
answers b queries in one device pass (kernels K8/K9 + copy-uncovered +
exact top-k) -- the reference has no batch API; column j of its result equals
``filter(dec, h, ys[j])``.

h is evaluated on the host exactly as the reference does (monotonicity
check, finiteness), only the r weights h(lambda) cross to the device.
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass
from typing import Callable, Sequence

import numpy as np

from . import _native as N
from .spectral import NumericalError, SpectralDecomposition, Variant

MONOTONICITY_SAMPLES = 1024
NORM_TOL = 1e-6


@dataclass(frozen=True)
class TransferFunction:
    """Scalar spectrum reshaping function with declared properties (``ranking.py:26-42``)."""

    fn: Callable[[np.ndarray], np.ndarray]
    nondecreasing: bool
    positive: bool
    name: str
    alpha: float | None = None
    analytic: bool = False

    def __call__(self, x) -> np.ndarray:
        return np.asarray(self.fn(np.asarray(x, dtype=np.float64)), dtype=np.float64)


def h_alpha(alpha: float) -> TransferFunction:
    """h(x) = (1 - alpha) / (1 - alpha x) (``ranking.py:45-65``)."""
    if not 0.0 <= alpha < 1.0:
        raise ValueError(f"alpha must lie in [0, 1), got {alpha}")

    def fn(x):
        return (1.0 - alpha) / (1.0 - alpha * x)

    return TransferFunction(fn=fn, nondecreasing=True, positive=True, name=f"h_alpha({alpha:g})", alpha=alpha,
                            analytic=True)


def custom_transfer(fn, nondecreasing: bool, positive: bool = False, name: str = "custom") -> TransferFunction:
    return TransferFunction(fn=fn, nondecreasing=nondecreasing, positive=positive, name=name)


def heat_kernel(t: float) -> TransferFunction:
    """exp(-t (1 - x)): nondecreasing, positive; sample-checked like any custom h."""
    return custom_transfer(lambda x: np.exp(-t * (1.0 - x)), nondecreasing=True, positive=True,
                           name=f"heat({t:g})")


def transfer_values(h: TransferFunction, eigenvalues: np.ndarray) -> np.ndarray:
    """h(Lambda) with the reference's checks (``ranking.py:77-102``)."""
    if not h.nondecreasing:
        raise ValueError(f"transfer function {h.name!r} is not declared nondecreasing; "
                         "truncated filtering would be unsound")
    eigenvalues = np.asarray(eigenvalues, dtype=np.float64)
    if not h.analytic and eigenvalues.size:
        lo, hi = float(eigenvalues.min()), float(eigenvalues.max())
        if hi > lo:
            samples = h(np.linspace(lo, hi, MONOTONICITY_SAMPLES))
            if np.any(np.diff(samples) < -1e-12):
                raise ValueError(f"transfer function {h.name!r} decreases on [{lo:g}, {hi:g}] "
                                 "despite being declared nondecreasing")
    values = h(eigenvalues)
    if not np.all(np.isfinite(values)):
        raise NumericalError(f"transfer function {h.name!r} is not finite on the spectrum")
    return values


_transfer_values = transfer_values


@dataclass(frozen=True, eq=False)
class ObservationVector:
    """Sparse nonnegative query signal y (``ranking.py:105-155``)."""

    size: int
    indices: np.ndarray
    values: np.ndarray
    cap: int

    def __post_init__(self):
        indices = np.asarray(self.indices, dtype=np.int64)
        values = np.asarray(self.values, dtype=np.float64)
        if indices.ndim != 1 or indices.shape != values.shape:
            raise ValueError("indices and values must be 1-D and equally long")
        if indices.size:
            if np.any(np.diff(indices) <= 0):
                raise ValueError("indices must be strictly increasing")
            if indices[0] < 0 or indices[-1] >= self.size:
                raise ValueError("indices out of range")
            if values.min() < 0.0:
                raise ValueError("values must be nonnegative")
        if indices.size > self.cap:
            raise ValueError(f"more than cap={self.cap} nonzeros")
        object.__setattr__(self, "indices", indices)
        object.__setattr__(self, "values", values)

    @classmethod
    def from_dense(cls, y, cap: int | None = None) -> "ObservationVector":
        y = np.asarray(y, dtype=np.float64)
        idx = np.flatnonzero(y)
        return cls(size=y.size, indices=idx, values=y[idx], cap=cap if cap is not None else max(idx.size, 1))

    @property
    def nnz(self) -> int:
        return self.indices.size

    @property
    def is_empty(self) -> bool:
        return self.indices.size == 0

    def to_dense(self) -> np.ndarray:
        out = np.zeros(self.size)
        out[self.indices] = self.values
        return out

    def dot(self, x) -> float:
        return float(self.values @ x[self.indices]) if self.nnz else 0.0


class QueryBatch:
    """b observation vectors in CSC form (y_ptr, y_idx, y_val) on the host."""

    def __init__(self, size: int, y_ptr, y_idx, y_val):
        self.size = int(size)
        self.y_ptr = np.ascontiguousarray(y_ptr, dtype=np.int64)
        self.y_idx = np.ascontiguousarray(y_idx, dtype=np.int64)
        self.y_val = np.ascontiguousarray(y_val, dtype=np.float64)
        if self.y_ptr.ndim != 1 or self.y_ptr.size < 2 or self.y_ptr[0] != 0:
            raise ValueError("y_ptr must start at 0 and hold b+1 offsets")
        if np.any(np.diff(self.y_ptr) < 0) or self.y_ptr[-1] != self.y_idx.size or self.y_idx.size != self.y_val.size:
            raise ValueError("inconsistent query batch")
        if self.y_idx.size and (self.y_idx.min() < 0 or self.y_idx.max() >= self.size):
            raise ValueError("indices out of range")

    @property
    def b(self) -> int:
        return self.y_ptr.size - 1

    @property
    def nbytes(self) -> int:
        return self.y_ptr.nbytes + self.y_idx.nbytes + self.y_val.nbytes

    @classmethod
    def from_vectors(cls, ys: Sequence[ObservationVector]) -> "QueryBatch":
        if not ys:
            raise ValueError("empty query batch")
        size = ys[0].size
        if any(y.size != size for y in ys):
            raise ValueError("observation vectors of different sizes")
        ptr = np.zeros(len(ys) + 1, dtype=np.int64)
        ptr[1:] = np.cumsum([y.nnz for y in ys])
        idx = np.concatenate([y.indices for y in ys]) if ptr[-1] else np.zeros(0, np.int64)
        val = np.concatenate([y.values for y in ys]) if ptr[-1] else np.zeros(0, np.float64)
        return cls(size, ptr, idx, val)

    def column(self, j: int) -> ObservationVector:
        s, e = self.y_ptr[j], self.y_ptr[j + 1]
        return ObservationVector(self.size, self.y_idx[s:e], self.y_val[s:e], cap=max(1, e - s))

    def split(self, parts: int, part: int) -> "QueryBatch":
        """Contiguous slice of the queries for one of ``parts`` ranks."""
        b = self.b
        lo, hi = (b * part) // parts, (b * (part + 1)) // parts
        s, e = self.y_ptr[lo], self.y_ptr[hi]
        return QueryBatch(self.size, self.y_ptr[lo:hi + 1] - s, self.y_idx[s:e], self.y_val[s:e])


class DeviceQueries:
    """A QueryBatch resident on the device (copied from pinned host memory)."""

    def __init__(self, batch: QueryBatch, dtype, device, non_blocking=True):
        import torch

        self.batch = batch
        self.b = batch.b
        pin = torch.cuda.is_available()

        def up(a, dt):
            t = torch.from_numpy(a)
            if pin:
                t = t.pin_memory()
            return t.to(device=device, dtype=dt, non_blocking=non_blocking)

        self.y_ptr = up(batch.y_ptr, torch.int64)
        self.y_idx = up(batch.y_idx, torch.int64)
        self.y_val = up(batch.y_val, dtype) if batch.y_val.size else torch.zeros(1, dtype=dtype, device=device)

    @property
    def h2d_bytes(self) -> int:
        return self.y_ptr.numel() * 8 + self.y_idx.numel() * 8 + self.y_val.numel() * self.y_val.element_size()


@dataclass
class FilterResult:
    """Device outputs of ``filter_batch``: X (b x n) and/or top-k (b x k)."""

    X: object = None
    top_idx: object = None
    top_val: object = None


def _weights_device(dec: SpectralDecomposition, h: TransferFunction):
    import torch

    key = (id(h), h.name)
    cache = dec.__dict__.setdefault("_w_cache", {})
    if key not in cache:
        w = transfer_values(h, dec.eigenvalues)
        cache[key] = (h, torch.as_tensor(w).to(device=dec.eta_device.device, dtype=dec.dtype))
    return cache[key][1]


def filter_device(dec: SpectralDecomposition, h: TransferFunction, queries: DeviceQueries,
                  copy_uncovered: bool | None = None, topk: int = 0, want_x: bool = True,
                  out: FilterResult | None = None, workspace=None) -> FilterResult:
    """All b queries through K8/K9 (+ copy-uncovered, + top-k) on the device."""
    import torch

    if queries.batch.size != dec.n:
        raise ValueError(f"observation size {queries.batch.size} != decomposition size {dec.n}")
    if copy_uncovered is None:
        copy_uncovered = dec.variant in (Variant.APPROX, Variant.SPARSE)
    w = _weights_device(dec, h)
    dev = dec.eta_device.device
    ctx = N.Context.get(dev)
    dt = dec.dtype
    dtc = N.dtype_code(dt)
    n, r, b = dec.n, dec.r, queries.b
    res = out or FilterResult()
    if want_x and res.X is None:
        res.X = torch.empty(b, n, dtype=dt, device=dev)
    if topk and res.top_idx is None:
        res.top_idx = torch.empty(b, topk, dtype=torch.int64, device=dev)
        res.top_val = torch.empty(b, topk, dtype=dt, device=dev)
    U = dec.U_device
    path = online_path(dec, b, topk if not want_x else 0, ctx)
    if path == "stream":
        packed = stream_layout(dec)
        need = int(ctx.lib.fsr_filter_stream_workspace_bytes(n, r, b))
        if workspace is None or workspace.numel() < need:
            workspace = torch.empty(need, dtype=torch.uint8, device=dev)
        ctx.call("filter_topk_stream", n, r, U.nnz, N.ptr(U.indptr), N.ptr(U.indices), N.ptr(U.values),
                 N.ptr(packed), N.ptr(w), N.ptr(dec.eta_device), b, N.ptr(queries.y_ptr), N.ptr(queries.y_idx),
                 N.ptr(queries.y_val), int(bool(copy_uncovered)), N.ptr(workspace), int(topk), N.ptr(res.top_idx),
                 N.ptr(res.top_val))
        ctx.last_online_path = "stream"
        return res
    if path == "tc":
        dense = dense_layout(dec)
        if dense is not None:
            need = int(ctx.lib.fsr_filter_tc_workspace_bytes(n, r, b))
            if workspace is None or workspace.numel() < need:
                workspace = torch.empty(need, dtype=torch.uint8, device=dev)
            ctx.call("filter_topk_tc", n, r, N.ptr(U.indptr), N.ptr(U.indices), N.ptr(U.values), N.ptr(dense),
                     N.ptr(w), N.ptr(dec.eta_device), b, N.ptr(queries.y_ptr), N.ptr(queries.y_idx),
                     N.ptr(queries.y_val), int(bool(copy_uncovered)), N.ptr(workspace), int(topk),
                     N.ptr(res.top_idx), N.ptr(res.top_val))
            ctx.last_online_path = "tc"
            return res
    need = int(ctx.lib.fsr_filter_workspace_bytes(dtc, n, r, b, int(not want_x)))
    if workspace is None or workspace.numel() < need:
        workspace = torch.empty(need, dtype=torch.uint8, device=dev)
    ctx.last_online_path = "pruned" if path != "exact" and topk_pruned(n, b, topk, dt) else "exact"
    if dec.is_sparse and dt == torch.float32 and ctx.single_query_path == "sell" and \
            (b == 1 or (b <= SELL_MAX_BATCH and r <= SELL_MAX_BATCH_RANK)):
        # up to 64 fp32 queries: K9e streams the sliced-ELL copy of U~ (6 bytes per entry, thread per
        # row, 1 / 2 / 4 queries per pass)
        sell = sell_layout(dec)
        if sell is not None:
            perm, lens, slice_ptr, scols, svals, n_long = sell
            ctx.call("filter_batch_sell", n, r, N.ptr(U.indptr), N.ptr(U.indices), N.ptr(u16_columns(dec)),
                     N.ptr(U.values), N.ptr(perm), N.ptr(lens), N.ptr(slice_ptr), N.ptr(scols), N.ptr(svals), n_long,
                     N.ptr(w), N.ptr(dec.eta_device), b, N.ptr(queries.y_ptr), N.ptr(queries.y_idx),
                     N.ptr(queries.y_val), int(bool(copy_uncovered)), N.ptr(workspace),
                     N.ptr(res.X if want_x else None), int(topk), N.ptr(res.top_idx if topk else None),
                     N.ptr(res.top_val if topk else None))
            ctx.last_online_path = "sell"
            return res
    if dec.is_sparse:
        # without the sliced-ELL copy a single fp32 query streams the CSR with 16-bit column indices
        c16 = u16_columns(dec) if b == 1 and dt == torch.float32 and r <= 65536 else None
        uargs = (1, N.ptr(U.indptr), N.ptr(U.indices), N.ptr(c16), N.ptr(U.values), N.ptr(None), 0)
    else:
        uargs = (0, N.ptr(None), N.ptr(None), N.ptr(None), N.ptr(None), N.ptr(U), U.stride(0))
    ctx.call("filter_batch_u16", dtc, n, r, *uargs, N.ptr(w), N.ptr(dec.eta_device), b, N.ptr(queries.y_ptr),
             N.ptr(queries.y_idx), N.ptr(queries.y_val), int(bool(copy_uncovered)), N.ptr(workspace),
             N.ptr(res.X if want_x else None), int(topk), N.ptr(res.top_idx if topk else None),
             N.ptr(res.top_val if topk else None))
    return res


def u16_columns(dec):
    """16-bit copy of U~'s column indices (r <= 65536), built once per
    decomposition and cached on it (fsr_u16_columns)."""
    import torch

    cached = getattr(dec, "_cols16", None)
    if cached is None:
        U = dec.U_device
        cached = torch.empty(max(1, U.nnz), dtype=torch.int16, device=U.indices.device)
        N.Context.get(U.indices.device).call("u16_columns", U.nnz, N.ptr(U.indices), N.ptr(cached))
        dec._cols16 = cached
    return cached


ONLINE_PATHS = ("tc", "stream", "pruned", "exact")  # last_online_path also reports "sell" (K9e, b <= 16)
# below this batch the tensor-core step (64-query tiles for b <= 64) streams
# the whole dense U~ for too few queries; the exact sparse K9 is faster there
# -- and, at C3, also faster than the packed-U~ stream K9s (opt-in:
# set_online_path("stream"))
TC_MIN_BATCH = 64


def online_path(dec, b: int, topk: int, ctx=None) -> str:
    """Which kernels a ``filter_device`` call runs: "tc" (top-k only, fp32
    sparse U~: K9t, the certified tensor-core step of csrc/k9t.cu, b >= 128),
    "stream" (K9s: the same certification on a packed fp16 U~ streamed from
    HBM; only when preferred), "pruned" (the certified fp16-gather K9h of
    csrc/prune.cuh), or "exact" (unpruned K9 + exact top-k).  The certified
    paths return the top-k of the unpruned sequential-order fp32 path bit for
    bit (for b <= 64 the exact path's narrow kernels sum rows in another
    order, see tests/test_gpu_prune.py).  The context's ``online_path``
    preference ("tc" by default) and the shape limits decide;
    ``set_topk_prune(False)`` forces "exact"."""
    import torch

    ctx = ctx or N.Context.get(dec.eta_device.device)
    if not topk or not dec.is_sparse or dec.dtype != torch.float32 or not ctx.topk_prune:
        return "exact"
    pref = ctx.online_path
    if pref == "tc" and b >= TC_MIN_BATCH and tc_pays(dec, b) and \
            ctx.lib.fsr_filter_tc_applicable(dec.n, dec.r, b, int(topk)):
        return "tc"
    if pref == "stream" and ctx.lib.fsr_filter_stream_applicable(dec.n, dec.r, dec.U_device.nnz, b, int(topk)):
        return "stream"
    if pref in ("tc", "pruned") and topk_pruned(dec.n, b, topk, dec.dtype):
        return "pruned"
    return "exact"


def tc_pays(dec, b: int) -> bool:
    """Cost model of K9t against the sparse K9 for a batch of b: the sparse
    kernel gathers 4 b bytes of Zs from L2 per nonzero of U~ (~12 TB/s
    measured), K9t streams the 2 n r byte dense fp16 U~ from HBM (~6.5 TB/s)
    whatever tau is.  C3, b = 64 measured: 1% exact 1.48 vs K9t 1.90 ms; 2%
    2.29 vs 1.96; 5% 4.8 vs 2.05 (the model's crossover: density 0.92 / b)."""
    return 4.0 * dec.U_device.nnz * b / 12.0 >= 2.0 * dec.n * dec.r / 6.5


def dense_layout(dec):
    """The fp16 dense copy of a float32 U~ (+ per-row bound factors) that the
    tensor-core step reads (fsr_dense_u_build), built once per decomposition
    and cached on it; None when the device lacks the memory (n x r x 2 bytes
    plus 2 GB of headroom), in which case the sparse paths run."""
    import torch

    cached = getattr(dec, "_dense_u", None)
    if cached is not None:
        return cached
    if getattr(dec, "_dense_u_failed", False):
        return None
    U = dec.U_device
    dev = dec.eta_device.device
    ctx = N.Context.get(dev)
    nbytes = int(ctx.lib.fsr_dense_u_bytes(dec.n, dec.r))
    free, _ = torch.cuda.mem_get_info(dev)
    if nbytes + (2 << 30) > free:
        torch.cuda.empty_cache()
        free, _ = torch.cuda.mem_get_info(dev)
        if nbytes + (2 << 30) > free:
            dec._dense_u_failed = True
            return None
    buf = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    ctx.call("dense_u_build", dec.n, dec.r, N.ptr(U.indptr), N.ptr(U.indices), N.ptr(U.values), N.ptr(buf))
    dec._dense_u = buf
    return buf


def stream_layout(dec):
    """The packed U~ (4 bytes per entry: fp16 value << 16 | column, per-row
    bound factors, chunk table) that the small-batch stream K9s reads
    (fsr_stream_u_build), built once per decomposition and cached on it."""
    import torch

    cached = getattr(dec, "_stream_u", None)
    if cached is not None:
        return cached
    U = dec.U_device
    dev = dec.eta_device.device
    ctx = N.Context.get(dev)
    buf = torch.empty(int(ctx.lib.fsr_stream_u_bytes(dec.n, dec.r, U.nnz)), dtype=torch.uint8, device=dev)
    ctx.call("stream_u_build", dec.n, dec.r, U.nnz, N.ptr(U.indptr), N.ptr(U.indices), N.ptr(U.values), N.ptr(buf))
    dec._stream_u = buf
    return buf


# Rows of U~ longer than the layout's long-row length stay in CSR (a warp per
# row).  None = chosen per decomposition: the smallest candidate whose long
# rows hold at most SELL_MAX_LONG_SHARE of the entries.  A slice w entries wide
# is one thread-per-row chain of w / 8 load round trips, so the widest slices
# bound the kernel when the stream itself is short (C3 1%: K9 0.094 ms at 512,
# 0.076 at 320), while the long rows' sequential chains run through warp
# shuffles (3 instructions per entry per warp) and pay only while they hold a
# small share of the entries: C3 5% needs 1024 (K9 0.259 ms against the CSR
# kernel's 0.329; at 512 a third of the entries are long: 0.9 ms).  Measured
# and not kept for the long rows: 32 or 8 rows per warp parked in shared
# memory with a thread per row's chain, on a side stream (one DRAM latency per
# 32/128 entries of a row: 0.55 / 0.21 ms at 2%, profiles/r02/k9e_long_rows.md).
SELL_LONG_ROW = None
SELL_LONG_ROW_CANDIDATES = (64, 96, 128, 192, 256, 320, 384, 448, 512, 640, 768, 1024, 1536, 2048)
SELL_MAX_RANK = 16384  # z must fit the SpMV's shared memory (fsr::sell::applicable)
SELL_MAX_LONG_SHARE = 0.03
# K9e with 2 / 4 queries per pass beats the CSR narrow kernels up to b = 16 (C3 2%: b = 8 0.44 vs
# 1.33 ms, b = 16 0.89 vs 1.34; b = 32 1.60 vs 1.35; 1%: b = 16 0.50 vs 0.86, b = 64 1.53 vs 1.24;
# profiles/r02/k9e_long_rows.md); libfsr accepts up to fsr::sell::kMaxBatch = 64
SELL_MAX_BATCH = 16
SELL_MAX_BATCH_RANK = 12800  # fsr::sell::batch_applicable


def sell_layout(dec):
    """The sliced-ELL copy of U~ that the single-query filter streams (K9e,
    csrc/k9e.cuh): rows sorted by length, 32-row slices stored column-major
    with 16-bit columns (fsr_sell_plan / fsr_sell_pack).  Built once per
    decomposition and cached on it; None when the layout does not apply
    (dense or fp64 U, r > 16384, a U~ without entries, or no long-row length
    up to 2048 whose longer rows hold at most SELL_MAX_LONG_SHARE of the
    entries)."""
    import ctypes
    import torch

    cached = dec.__dict__.get("_sell_u", False)
    if cached is not False:
        return cached
    dec._sell_u = None
    if not dec.is_sparse or dec.dtype != torch.float32 or dec.r > SELL_MAX_RANK or dec.U_device.nnz == 0:
        return None
    U = dec.U_device
    dev = U.indices.device
    row_len = U.indptr[1:] - U.indptr[:-1]
    long_row = None
    for cand in ((SELL_LONG_ROW,) if SELL_LONG_ROW else SELL_LONG_ROW_CANDIDATES):
        if float(row_len[row_len > cand].sum()) <= SELL_MAX_LONG_SHARE * U.nnz:
            long_row = int(cand)
            break
    del row_len
    if long_row is None:
        return None  # the CSR single-query kernel serves this U~
    ctx = N.Context.get(dev)
    n = dec.n
    ws = torch.empty(int(ctx.lib.fsr_sell_plan_workspace_bytes(n)), dtype=torch.uint8, device=dev)
    perm = torch.empty(n, dtype=torch.int32, device=dev)
    lens = torch.empty(n, dtype=torch.int32, device=dev)
    slice_ptr = torch.empty((n + 31) // 32 + 1, dtype=torch.int64, device=dev)
    n_long, total = ctypes.c_int64(0), ctypes.c_int64(0)
    ctx.call("sell_plan", n, N.ptr(U.indptr), long_row, N.ptr(perm), N.ptr(lens), N.ptr(slice_ptr), N.ptr(ws),
             ctypes.byref(n_long), ctypes.byref(total))
    del ws
    cols = torch.empty(max(1, total.value), dtype=torch.int16, device=dev)
    vals = torch.empty(max(1, total.value), dtype=torch.float32, device=dev)
    ctx.call("sell_pack", n, N.ptr(U.indptr), N.ptr(U.indices), N.ptr(U.values), N.ptr(perm), N.ptr(slice_ptr),
             N.ptr(cols), N.ptr(vals))
    dec._sell_u = (perm, lens, slice_ptr, cols, vals, int(n_long.value))
    return dec._sell_u


def last_fallback_count(workspace, dec, b: int, ctx=None) -> int:
    """Queries of the last certified call (tc or pruned) that went through the
    exact fallback."""
    import ctypes

    ctx = ctx or N.Context.get(dec.eta_device.device)
    if ctx.last_online_path in ("tc", "stream"):
        out = ctypes.c_int()
        ctx.call("filter_tc_fallback_count", N.ptr(workspace), ctypes.byref(out))
        return int(out.value)
    return pruned_fallback_count(workspace, dec.n, dec.r, b)


def last_tc_stats(workspace, dec, b: int):
    """(candidate rows, rows re-scored exactly) per query of the last
    tensor-core call, as an int32 array (b x 2)."""
    ctx = N.Context.get(dec.eta_device.device)
    out = np.zeros((b, 2), dtype=np.int32)
    ctx.call("filter_tc_stats", dec.n, dec.r, b, N.ptr(workspace), out.ctypes.data)
    return out


def filter_workspace_bytes(dec, b: int, want_x: bool, topk: int = 0) -> int:
    """Workspace bytes ``filter_device`` needs for this call's path."""
    ctx = N.Context.get(dec.eta_device.device)
    need = int(ctx.lib.fsr_filter_workspace_bytes(N.dtype_code(dec.dtype), dec.n, dec.r, b, int(not want_x)))
    path = online_path(dec, b, topk, ctx) if not want_x else "exact"
    if path == "tc":
        need = max(need, int(ctx.lib.fsr_filter_tc_workspace_bytes(dec.n, dec.r, b)))
    elif path == "stream":
        need = max(need, int(ctx.lib.fsr_filter_stream_workspace_bytes(dec.n, dec.r, b)))
    return need


def topk_pruned(n: int, b: int, k: int, dtype, sparse: bool = True) -> bool:
    """Whether a top-k-only ``filter_device`` call takes the certified pruned
    path (csrc/prune.cuh ``applicable``; the context option FSR_OPT_TOPK_PRUNE
    must also be on): fp32 sparse U~, n >= 131072, b >= 256, b % 8 == 0,
    1 <= k <= 256 (csrc/prune.cuh `applicable`).  Its top-k equals the unpruned fp32 path's bit for bit."""
    import torch

    return (sparse and dtype == torch.float32 and 131072 <= n < 2 ** 31 and b >= 256 and b % 8 == 0
            and 1 <= k <= 256)


def pruned_fallback_count(workspace, n: int, r: int, b: int) -> int:
    """Queries of the last pruned call answered by the exact fallback (the
    counter in filter_pruned's workspace layout, csrc/k8_online.cu)."""
    import torch

    al = lambda x: (x + 255) // 256 * 256  # noqa: E731
    off = al(b * r * 4) + al(r * b * 4) + al(n * b * 4) + al(r * b * 2) + al(b * 8) + al(n * 4)
    return int(workspace[off:off + 4].view(torch.int32).item())


def _as_device_dec(dec) -> SpectralDecomposition:
    if isinstance(dec, SpectralDecomposition):
        return dec
    cache = getattr(_as_device_dec, "_cache", None)
    if cache is None:
        cache = _as_device_dec._cache = {}
    hit = cache.get(id(dec))
    if hit is None or hit[0] is not dec:
        hit = cache[id(dec)] = (dec, SpectralDecomposition.from_host(dec))
    return hit[1]


def filter(dec, h: TransferFunction, y: ObservationVector, copy_uncovered: bool | None = None) -> np.ndarray:
    """x = U h(Lambda) U^T y (``ranking.py:229-255``) for one query, on the device."""
    dec = _as_device_dec(dec)
    if y.size != dec.n:
        raise ValueError(f"observation size {y.size} != decomposition size {dec.n}")
    return filter_batch(dec, h, [y], copy_uncovered=copy_uncovered)[0]


def filter_batch(dec, h: TransferFunction, ys, copy_uncovered: bool | None = None, topk: int | None = None):
    """Batched ``filter``: rows of the returned (b x n) array are the score
    vectors of ``ys`` (a list of ObservationVector or a QueryBatch).  With
    ``topk`` returns (top_idx, top_val) host arrays (b x topk) in ``rank``
    order instead of the scores."""
    import torch

    dec = _as_device_dec(dec)
    batch = ys if isinstance(ys, QueryBatch) else QueryBatch.from_vectors(list(ys))
    if batch.size != dec.n:
        raise ValueError(f"observation size {batch.size} != decomposition size {dec.n}")
    q = DeviceQueries(batch, dec.dtype, dec.eta_device.device)
    res = filter_device(dec, h, q, copy_uncovered=copy_uncovered, topk=topk or 0, want_x=not topk)
    torch.cuda.current_stream(dec.eta_device.device).synchronize()
    if topk:
        return res.top_idx.cpu().numpy(), res.top_val.double().cpu().numpy()
    return res.X.double().cpu().numpy()


def rank(x_pooled) -> np.ndarray:
    """Indices by descending score, ties by ascending index (``ranking.py:390-395``)."""
    x_pooled = np.asarray(x_pooled, dtype=np.float64)
    if not np.all(np.isfinite(x_pooled)):
        raise NumericalError("scores contain NaN or infinity")
    return np.lexsort((np.arange(x_pooled.size), -x_pooled)).astype(np.int64)


def top_k(dec, h: TransferFunction, ys, k: int = 100, copy_uncovered: bool | None = None):
    """First k entries of ``rank(filter(dec, h, y))`` for every query, on the device."""
    return filter_batch(dec, h, ys, copy_uncovered=copy_uncovered, topk=k)


def empty_query_warning(y: ObservationVector) -> None:
    if y.is_empty:
        warnings.warn("query has no positive similarity to the dataset; empty observation")


# ---------------------------------------------------------------------------
# Epilogues around the online path (reference ranking.py:256-411, SURVEY.md
# 8(f) row 3): FSRw, region->image pooling, the explicit embedding.  Device
# kernels K10 (csrc/k10_epilogue.cu) and the K8 projection.
# ---------------------------------------------------------------------------

def _check_query_regions(query_regions, d: int) -> np.ndarray:
    """Same validation as the reference (``ranking.py:156-165``)."""
    regions = np.atleast_2d(np.asarray(query_regions, dtype=np.float64))
    if regions.size == 0:
        raise ValueError("query must contain at least one region vector")
    if regions.shape[1] != d:
        raise ValueError(f"query dimension {regions.shape[1]} != dataset dimension {d}")
    norms = np.linalg.norm(regions, axis=1)
    if np.any(np.abs(norms - 1.0) > NORM_TOL):
        raise ValueError("query vectors must be unit-norm")
    return regions


def _host_vectors(data) -> np.ndarray:
    """Dataset vectors of a reference ``DescriptorSet`` (``.vectors``) or an array."""
    v = getattr(data, "vectors", data)
    if hasattr(v, "detach"):
        return v
    return np.asarray(v, dtype=np.float64)


def _device_vectors(data, dtype, device):
    import torch

    v = _host_vectors(data)
    if hasattr(v, "detach"):
        return v.to(device=device, dtype=dtype).contiguous()
    cache = _device_vectors.__dict__.setdefault("_cache", {})
    key = (id(data), dtype, str(device))
    hit = cache.get(key)
    if hit is None or hit[0] is not data:
        hit = cache[key] = (data, torch.as_tensor(v).to(device=device, dtype=dtype).contiguous())
    return hit[1]


def fsrw_correct_device(X, dec: SpectralDecomposition, V, Qsum):
    """In place: X[j] += (1 - eta) * (V Qsum[j]) for the (b x n) device scores X."""
    ctx = N.Context.get(X.device)
    b, n = X.shape
    if V.shape[0] != n or dec.n != n or Qsum.shape != (b, V.shape[1]):
        raise ValueError("score rows, dataset and decomposition sizes must agree")
    ctx.call("fsrw_correct", N.dtype_code(X.dtype), b, n, V.shape[1], N.ptr(V), V.stride(0), N.ptr(Qsum),
             Qsum.stride(0), N.ptr(dec.eta_device), N.ptr(X), X.stride(0))
    return X


def fsrw_correct(x, dec, data, query_regions) -> np.ndarray:
    """x + (1 - eta) * (V . sum of query regions) (``ranking.py:256-274``), on the device."""
    import torch

    dec = _as_device_dec(dec)
    V_host = _host_vectors(data)
    n, d = V_host.shape
    regions = _check_query_regions(query_regions, d)
    x = np.asarray(x, dtype=np.float64)
    if x.shape != (n,) or dec.n != n:
        raise ValueError("score vector, dataset and decomposition sizes must agree")
    dev = dec.eta_device.device
    V = _device_vectors(data, dec.dtype, dev)
    X = torch.as_tensor(x).to(device=dev, dtype=dec.dtype).reshape(1, n).contiguous()
    Qs = torch.as_tensor(regions.sum(axis=0)).to(device=dev, dtype=dec.dtype).reshape(1, d)
    fsrw_correct_device(X, dec, V, Qs)
    return X[0].double().cpu().numpy()


@dataclass(frozen=True, eq=False)
class PoolingMatrix:
    """Sparse (N, n) region->image map (``ranking.py:277-319``): every region
    column owned by exactly one image row, finite nonnegative weights."""

    csr: object

    def __post_init__(self):
        import scipy.sparse as sp

        mat = sp.csr_matrix(self.csr, dtype=np.float64)
        counts = np.asarray((mat != 0).sum(axis=0)).ravel()
        if np.any(counts != 1):
            raise ValueError("each region must belong to exactly one image")
        if not np.all(np.isfinite(mat.data)) or (mat.nnz and mat.data.min() < 0.0):
            raise ValueError("pooling weights must be finite and nonnegative")
        object.__setattr__(self, "csr", mat)

    @classmethod
    def identity(cls, n: int) -> "PoolingMatrix":
        import scipy.sparse as sp

        return cls(sp.identity(n, dtype=np.float64, format="csr"))

    @classmethod
    def from_region_map(cls, region_to_image, n_images: int | None = None, weights=None) -> "PoolingMatrix":
        import scipy.sparse as sp

        r2i = np.asarray(region_to_image, dtype=np.int64)
        n = r2i.size
        n_images = int(r2i.max()) + 1 if n_images is None else n_images
        data = np.ones(n) if weights is None else np.asarray(weights, dtype=np.float64)
        return cls(sp.csr_matrix((data, (r2i, np.arange(n))), shape=(n_images, n)))

    @property
    def n_images(self) -> int:
        return self.csr.shape[0]

    @property
    def n_regions(self) -> int:
        return self.csr.shape[1]

    def device(self, dtype, device):
        """(indptr int64, indices int32, values dtype) of the CSR on the device (cached)."""
        import torch

        cache = self.__dict__.setdefault("_dev", {})
        key = (dtype, str(device))
        if key not in cache:
            m = self.csr
            m.sort_indices()
            cache[key] = (torch.as_tensor(m.indptr.astype(np.int64)).to(device),
                          torch.as_tensor(m.indices.astype(np.int32)).to(device),
                          torch.as_tensor(m.data).to(device=device, dtype=dtype))
        return cache[key]


def pool_device(pooling: PoolingMatrix, X):
    """(b x N) image scores of the (b x n_regions) device scores X."""
    import torch

    b, n = X.shape
    if n != pooling.n_regions:
        raise ValueError(f"score vector length {n} != {pooling.n_regions} regions")
    ip, ix, pv = pooling.device(X.dtype, X.device)
    out = torch.empty(b, pooling.n_images, dtype=X.dtype, device=X.device)
    N.Context.get(X.device).call("pool_scores", N.dtype_code(X.dtype), b, pooling.n_images, N.ptr(ip), N.ptr(ix),
                                 N.ptr(pv), N.ptr(X), X.stride(0), N.ptr(out), out.stride(0))
    return out


def pool(pooling: PoolingMatrix, x) -> np.ndarray:
    """Image scores P x (``ranking.py:322-326``), on the device."""
    import torch

    x = np.asarray(x, dtype=np.float64)
    if x.shape != (pooling.n_regions,):
        raise ValueError(f"score vector length {x.shape} != {pooling.n_regions} regions")
    dev = torch.device("cuda", torch.cuda.current_device())
    X = torch.as_tensor(x).to(dev).reshape(1, -1)
    return pool_device(pooling, X)[0].cpu().numpy()


def pooled_basis_device(pooling: PoolingMatrix, dec: SpectralDecomposition):
    """U_bar = P U (N x r) on the device (``ranking.py:329-334``)."""
    import torch

    if pooling.n_regions != dec.n:
        raise ValueError("pooling width does not match the decomposition")
    dev = dec.eta_device.device
    ip, ix, pv = pooling.device(dec.dtype, dev)
    Ub = torch.empty(pooling.n_images, dec.r, dtype=dec.dtype, device=dev)
    U = dec.U_device
    if dec.is_sparse:
        uargs = (1, N.ptr(U.indptr), N.ptr(U.indices), N.ptr(U.values), N.ptr(None), 0)
    else:
        uargs = (0, N.ptr(None), N.ptr(None), N.ptr(None), N.ptr(U), U.stride(0))
    N.Context.get(dev).call("pool_rows", N.dtype_code(dec.dtype), pooling.n_images, N.ptr(ip), N.ptr(ix), N.ptr(pv),
                            dec.n, dec.r, *uargs, N.ptr(Ub), Ub.stride(0))
    return Ub


def pooled_basis(pooling: PoolingMatrix, dec) -> np.ndarray:
    """Precomputed (N, r) pooled basis (``ranking.py:329-334``), as a host array."""
    dec = _as_device_dec(dec)
    return pooled_basis_device(pooling, dec).double().cpu().numpy()


def _project_device(dec: SpectralDecomposition, w, queries: DeviceQueries):
    import torch

    dev = dec.eta_device.device
    Zt = torch.empty(queries.b, dec.r, dtype=dec.dtype, device=dev)
    U = dec.U_device
    if dec.is_sparse:
        uargs = (1, N.ptr(U.indptr), N.ptr(U.indices), N.ptr(U.values), N.ptr(None), 0)
    else:
        uargs = (0, N.ptr(None), N.ptr(None), N.ptr(None), N.ptr(U), U.stride(0))
    N.Context.get(dev).call("project_batch", N.dtype_code(dec.dtype), dec.n, dec.r, *uargs, N.ptr(w), queries.b,
                            N.ptr(queries.y_ptr), N.ptr(queries.y_idx), N.ptr(queries.y_val), N.ptr(Zt))
    return Zt


def filter_pooled_device(dec: SpectralDecomposition, h: TransferFunction, queries: DeviceQueries, U_bar):
    """(b x N) image scores U_bar h(Lambda) U^T y_j; no uncovered copy (``ranking.py:337-353``)."""
    import torch

    if queries.batch.size != dec.n:
        raise ValueError(f"observation size {queries.batch.size} != decomposition size {dec.n}")
    if U_bar.shape[1] != dec.r:
        raise ValueError("pooled basis width does not match the decomposition")
    Zt = _project_device(dec, _weights_device(dec, h), queries)
    out = torch.empty(queries.b, U_bar.shape[0], dtype=dec.dtype, device=Zt.device)
    N.Context.get(Zt.device).call("dense_scores", N.dtype_code(dec.dtype), U_bar.shape[0], dec.r, N.ptr(U_bar),
                                  U_bar.stride(0), queries.b, N.ptr(Zt), Zt.stride(0), N.ptr(out), out.stride(0))
    return out


def filter_pooled(dec, h: TransferFunction, y: ObservationVector, U_bar) -> np.ndarray:
    """Image scores directly, U_bar h(Lambda) U^T y (``ranking.py:337-353``), on the device."""
    import torch

    dec = _as_device_dec(dec)
    if y.size != dec.n:
        raise ValueError(f"observation size {y.size} != decomposition size {dec.n}")
    dev = dec.eta_device.device
    Ub = U_bar if hasattr(U_bar, "detach") else torch.as_tensor(np.asarray(U_bar, dtype=np.float64))
    Ub = Ub.to(device=dev, dtype=dec.dtype).contiguous()
    q = DeviceQueries(QueryBatch.from_vectors([y]), dec.dtype, dev)
    return filter_pooled_device(dec, h, q, Ub)[0].double().cpu().numpy()


@dataclass(frozen=True, eq=False)
class RankingResult:
    """Region scores, pooled image scores and the image order (``ranking.py:398-411``)."""

    x: np.ndarray
    x_pooled: np.ndarray
    order: np.ndarray

    @classmethod
    def from_scores(cls, x, pooling: PoolingMatrix | None = None) -> "RankingResult":
        x = np.asarray(x, dtype=np.float64)
        x_pooled = pool(pooling, x) if pooling is not None else x
        return cls(x=x, x_pooled=x_pooled, order=rank(x_pooled))


class Embedding:
    """Phi = h(Lambda)^{1/2} U^T (``ranking.py:356-365``) bound to a device
    decomposition: ``phi @ psi`` runs the K8 projection with weights sqrt(w);
    ``matrix()`` materialises the reference's object (scipy CSR or ndarray)."""

    def __init__(self, dec: SpectralDecomposition, h: TransferFunction):
        import torch

        w = transfer_values(h, dec.eigenvalues)
        if np.any(w < 0.0):
            raise ValueError("transfer values must be nonnegative to take a square root")
        self.dec = dec
        self.scale = np.sqrt(w)
        self.scale_device = torch.as_tensor(self.scale).to(device=dec.eta_device.device, dtype=dec.dtype)

    @property
    def shape(self):
        return (self.dec.r, self.dec.n)

    def __matmul__(self, psi) -> np.ndarray:
        y = psi if isinstance(psi, ObservationVector) else ObservationVector.from_dense(psi)
        if y.size != self.dec.n:
            raise ValueError(f"vector size {y.size} != {self.dec.n}")
        q = DeviceQueries(QueryBatch.from_vectors([y]), self.dec.dtype, self.dec.eta_device.device)
        return _project_device(self.dec, self.scale_device, q)[0].double().cpu().numpy()

    def matrix(self):
        import scipy.sparse as sp

        if self.dec.is_sparse:
            U = self.dec.U_device
            vals = (U.values.double() * self.scale_device.double()[U.indices.long()]).cpu().numpy()
            m = sp.csr_matrix((vals, U.indices.cpu().numpy(), U.indptr.cpu().numpy()), shape=(self.dec.n, self.dec.r))
            return m.T.tocsr()
        U = self.dec.U_device.double() * self.scale_device.double()[None, :]
        return U.T.contiguous().cpu().numpy()


def embedding(dec, h: TransferFunction) -> Embedding:
    """Explicit feature map Phi = h(Lambda)^{1/2} U^T (``ranking.py:356-365``)."""
    return Embedding(_as_device_dec(dec), h)


def out_of_sample_similarity(z1, z2, phi, data, k: int, gamma: float) -> float:
    """(Phi psi(z1)) . (Phi psi(z2)) with psi(z)_i = s(v_i | z) on the k-NN of z
    (``ranking.py:368-387``); psi on the device (knn.observation_batch_device)."""
    import torch

    from .knn import observation_batch_device

    V_host = _host_vectors(data)
    n = V_host.shape[0]
    if k < 1 or k > n:
        raise ValueError(f"k must lie in [1, n], got {k}")
    if gamma <= 0:
        raise ValueError("gamma must be positive")
    dev = phi.dec.eta_device.device if isinstance(phi, Embedding) else torch.device("cuda", torch.cuda.current_device())
    V = _device_vectors(data, torch.float64, dev)
    Z = torch.as_tensor(np.stack([np.asarray(z1, dtype=np.float64), np.asarray(z2, dtype=np.float64)])).to(dev)
    ptr, idx, val = observation_batch_device(Z, V, k, gamma, cap=k)
    psis = [ObservationVector(n, idx[ptr[j]:ptr[j + 1]], val[ptr[j]:ptr[j + 1]], cap=max(1, k)) for j in (0, 1)]
    e1 = np.asarray(phi @ psis[0] if isinstance(phi, Embedding) else phi @ psis[0].to_dense()).ravel()
    e2 = np.asarray(phi @ psis[1] if isinstance(phi, Embedding) else phi @ psis[1].to_dense()).ravel()
    return float(e1 @ e2)


# ---------------------------------------------------------------------------
# CUDA-graph replay of the online step (small batches are launch-bound)
# ---------------------------------------------------------------------------

class _StaticQueries:
    """DeviceQueries-shaped view of fixed device buffers (graph-capturable)."""

    def __init__(self, size, b, y_ptr, y_idx, y_val):
        self.batch = QueryBatch(size, np.zeros(b + 1, np.int64), np.zeros(0, np.int64), np.zeros(0))
        self.b = b
        self.y_ptr, self.y_idx, self.y_val = y_ptr, y_idx, y_val


class FilterGraph:
    """One CUDA graph for ``filter_device`` over a fixed query capacity.

    The graph holds the pinned-host -> device copies of (y_ptr, y_idx,
    y_val), K8 projection, K9, copy-uncovered and the exact top-k; ``run``
    only refreshes the pinned staging buffers and replays it, so a query
    batch costs one graph launch instead of ~6 kernel launches and the
    Python/ctypes work between them.  Batches smaller than ``b`` are padded
    with empty queries.  Results are identical to ``filter_device`` called
    with a batch of the graph's capacity ``b`` (same kernels, same
    arguments); the kernel path is chosen by ``b``.  For a float32 sparse
    decomposition b <= 16 (K9e) and b >= 256 sum every row in CSR order, so
    their scores agree bit for bit; a partial batch run eagerly through
    ``filter_device`` with 17 <= b <= 64 queries may take the narrow CSR
    kernel (a row summed in two interleaved halves) and differ in the last
    bits of ``top_val`` and in the order of near-ties.
    """

    def __init__(self, dec: SpectralDecomposition, h: TransferFunction, b: int, nnz_cap: int, topk: int = 100,
                 copy_uncovered: bool | None = None):
        import torch

        if b < 1 or nnz_cap < 0 or topk < 1:
            raise ValueError("need b >= 1, nnz_cap >= 0, topk >= 1")
        self.dec, self.h, self.b, self.nnz_cap, self.topk = dec, h, b, nnz_cap, topk
        dev = dec.eta_device.device
        dt = dec.dtype
        cap = max(1, nnz_cap)
        # (y_ptr, y_idx, y_val) share one pinned staging buffer and one device buffer, so the
        # graph holds a single H2D copy node instead of three
        es = torch.empty(0, dtype=dt).element_size()
        o_idx = -(-(b + 1) * 8 // 256) * 256
        o_val = o_idx + -(-cap * 8 // 256) * 256
        total = o_val + -(-cap * es // 256) * 256
        self.h_all = torch.zeros(total, dtype=torch.uint8).pin_memory()
        self.d_all = torch.zeros(total, dtype=torch.uint8, device=dev)

        def views(buf):
            return (buf[: (b + 1) * 8].view(torch.int64), buf[o_idx: o_idx + cap * 8].view(torch.int64),
                    buf[o_val: o_val + cap * es].view(dt))

        self.h_ptr, self.h_idx, self.h_val = views(self.h_all)
        self.d_ptr, self.d_idx, self.d_val = views(self.d_all)
        self.queries = _StaticQueries(dec.n, b, self.d_ptr, self.d_idx, self.d_val)
        self.res = FilterResult(top_idx=torch.empty(b, topk, dtype=torch.int64, device=dev),
                                top_val=torch.empty(b, topk, dtype=dt, device=dev))
        ctx = N.Context.get(dev)
        self.ws = torch.empty(filter_workspace_bytes(dec, b, want_x=False, topk=topk), dtype=torch.uint8, device=dev)
        self.copy_uncovered = copy_uncovered
        self._done = None
        _weights_device(dec, h)  # cache h(Lambda) on the device before capture
        timing = bool(getattr(ctx, "_timing", False))
        side = torch.cuda.Stream(dev)
        side.wait_stream(torch.cuda.current_stream(dev))
        with torch.cuda.stream(side):  # warm-up: sizes libfsr scratch, sets kernel attributes
            for _ in range(2):
                self._body()
        torch.cuda.current_stream(dev).wait_stream(side)
        torch.cuda.synchronize(dev)
        ctx.enable_timing(False)
        self.graph = torch.cuda.CUDAGraph()
        try:
            with torch.cuda.graph(self.graph, stream=side):
                self._body()
        finally:
            ctx.enable_timing(timing)
            N.Context.get(dev)  # re-bind libfsr to the current stream

    def _body(self):
        self.d_all.copy_(self.h_all, non_blocking=True)
        filter_device(self.dec, self.h, self.queries, copy_uncovered=self.copy_uncovered, topk=self.topk,
                      want_x=False, out=self.res, workspace=self.ws)

    def stage(self, batch: QueryBatch) -> None:
        """Copy a host batch into the pinned staging buffers (host-only work;
        waits until the previous replay has consumed them)."""
        if self._done is not None:
            self._done.synchronize()
        if batch.size != self.dec.n:
            raise ValueError(f"observation size {batch.size} != decomposition size {self.dec.n}")
        if batch.b > self.b or int(batch.y_ptr[-1]) > self.nnz_cap:
            raise ValueError(f"batch ({batch.b} queries, {int(batch.y_ptr[-1])} nonzeros) exceeds the graph's "
                             f"capacity ({self.b}, {self.nnz_cap})")
        ptr = self.h_ptr.numpy()
        ptr[: batch.b + 1] = batch.y_ptr
        ptr[batch.b + 1:] = batch.y_ptr[-1]
        nz = int(batch.y_ptr[-1])
        self.h_idx.numpy()[:nz] = batch.y_idx
        self.h_val[:nz] = torch_from_numpy_cast(batch.y_val, self.h_val.dtype)

    def replay(self):
        """Launch the captured step on the current stream (after ``stage``)."""
        import torch

        self.graph.replay()
        self._done = torch.cuda.Event()
        self._done.record()
        return self.res

    def run(self, batch: QueryBatch):
        """stage + replay; returns the device FilterResult (top_idx / top_val, b x topk)."""
        self.stage(batch)
        return self.replay()

    def submit(self, batch: QueryBatch):
        """Asynchronous step: stage, replay and start the top-k D2H into pinned
        host buffers; ``fetch`` returns them.  Alternating two FilterGraphs
        overlaps one batch's host work with the other's device work."""
        import torch

        if not hasattr(self, "_h_idx"):
            self._h_idx = torch.empty(self.res.top_idx.shape, dtype=torch.int64).pin_memory()
            self._h_val = torch.empty(self.res.top_val.shape, dtype=self.res.top_val.dtype).pin_memory()
        self.run(batch)
        self._h_idx.copy_(self.res.top_idx, non_blocking=True)
        self._h_val.copy_(self.res.top_val, non_blocking=True)
        self._fetched = torch.cuda.Event()
        self._fetched.record()
        self._done = self._fetched  # staging buffers are reusable once the copies are done too
        self._nb = batch.b

    def fetch(self):
        """Wait for the last ``submit`` and return host (top_idx, top_val) of its
        queries as fresh arrays (the pinned buffers are overwritten by the
        next ``submit`` on this graph)."""
        self._fetched.synchronize()
        return self._h_idx[: self._nb].numpy().copy(), self._h_val[: self._nb].numpy().copy()


def torch_from_numpy_cast(a, dtype):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(dtype)
