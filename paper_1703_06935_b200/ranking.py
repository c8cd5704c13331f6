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
    need = int(ctx.lib.fsr_filter_workspace_bytes(dtc, n, r, b, int(not want_x)))
    if workspace is None or workspace.numel() < need:
        workspace = torch.empty(need, dtype=torch.uint8, device=dev)
    U = dec.U_device
    if dec.is_sparse:
        uargs = (1, N.ptr(U.indptr), N.ptr(U.indices), N.ptr(U.values), N.ptr(None), 0)
    else:
        uargs = (0, N.ptr(None), N.ptr(None), N.ptr(None), N.ptr(U), U.stride(0))
    ctx.call("filter_batch", dtc, n, r, *uargs, N.ptr(w), N.ptr(dec.eta_device), b, N.ptr(queries.y_ptr),
             N.ptr(queries.y_idx), N.ptr(queries.y_val), int(bool(copy_uncovered)), N.ptr(workspace),
             N.ptr(res.X if want_x else None), int(topk), N.ptr(res.top_idx if topk else None),
             N.ptr(res.top_val if topk else None))
    return res


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
