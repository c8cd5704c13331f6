"""Offline FSR on the device: range finder, Rayleigh-Ritz, sparsification.

Drop-in for the reference ``spectral`` module (``spectral.py``): the same
function names, argument meaning, defaults, validation errors and result
types; the arithmetic runs in libfsr (include/fsr.h) on a CUDA device.

Precision: ``dtype="float64"`` (default, the reference's precision -- "parity
mode") keeps every n x r_hat block in fp64.  ``dtype="float32"`` stores the
blocks and runs the SpMM in fp32 while Gram, projection, Cholesky and the
eigensolve stay fp64 ("fast mode").

Device residency: ``RangeBasis.Q/B`` and ``SpectralDecomposition.U`` are
torch CUDA tensors (``U_device``); ``SpectralDecomposition.U`` / ``.eta``
materialise host numpy/scipy copies only when touched.
"""

from __future__ import annotations

import enum
import math
import os
from dataclasses import dataclass, replace

import numpy as np
import scipy.sparse as sp

from . import _native as N
from .graph import ComponentLabeling
from .sparsemat import DeviceCSR, SparseSymmetricMatrix

DEFAULT_OVERSAMPLING = 10
DEFAULT_POWER_ITERATIONS = 4
DENSE_GUARD = 4096

# re-orthogonalisation trigger of spectral.py:167 (fp64); fp32 blocks cannot
# be orthonormal beyond ~1e-7, so their trigger is scaled accordingly.
ORTH_TOL = {N.F64: 1e-8, N.F32: 1e-4}
# CholeskyQR2 is orthogonal to O(eps) when the second Gram is this close to I
# (Yamamoto et al. 2015); beyond it an explicit check runs (spectral.py:167).
CHOLQR2_SAFE = 0.1
# first CholeskyQR pass of a float32 block with a one-slice Gram and a one-slice
# R^-1 (see _cholqr_pass / fsr_apply_rinv_levels)
FAST_FIRST_GRAM = True
FAST_FIRST_APPLY = os.environ.get("FSR_FAST_FIRST_APPLY", "1") != "0"
# float32 simultaneous iteration: intermediate rounds keep a well-conditioned
# basis (max|Q^T Q - I| <= PRECOND_TOL) instead of an orthonormal one; see range_finder
SI_SPAN_ONLY = os.environ.get("FSR_SI_SPAN_ONLY", "1") != "0"
PRECOND_TOL = 0.25
# decompose (fp32): the last round is preconditioned too and Rayleigh-Ritz
# solves the generalised problem with G = Q^T Q (see _rayleigh_ritz)
FUSED_RR = os.environ.get("FSR_FUSED_RR", "1") != "0"

_MASK64 = (1 << 64) - 1


class NumericalError(RuntimeError):
    """A computation left its supported regime (guards, non-finite values)."""


class Variant(str, enum.Enum):
    EXACT = "exact"
    RANK_R = "rank_r"
    APPROX = "approx"
    SPARSE = "sparse"


@dataclass(frozen=True)
class Provenance:
    r: int | None = None
    p: int | None = None
    q: int | None = None
    tau: int | None = None
    seed: int | None = None


@dataclass(frozen=True, eq=False)
class RangeBasis:
    """Q orthonormal (n x r_hat) and B = A Q, as device tensors."""

    Q: object
    B: object
    iterations_used: int
    seed: int | None = None

    @property
    def r_hat(self) -> int:
        return int(self.Q.shape[1])


class SpectralDecomposition:
    """Rank-r eigenpair approximation U diag(eigenvalues) U^T of A.

    ``U_device`` is a dense CUDA tensor (n x r) or a ``DeviceCSR`` after
    sparsification; ``eta_device`` the float64 row norms on the device.  The
    reference-facing attributes ``U`` (numpy / scipy CSR, float64) and ``eta``
    are host copies made on first access.
    """

    def __init__(self, U_device, eigenvalues, eta_device, components, variant, provenance):
        self.U_device = U_device
        self.eigenvalues = np.asarray(eigenvalues, dtype=np.float64)
        self.eta_device = eta_device
        self.components = components
        self.variant = Variant(variant)
        self.provenance = provenance
        self._U_host = None
        self._eta_host = None

    @property
    def n(self) -> int:
        return int(self.U_device.shape[0])

    @property
    def r(self) -> int:
        return int(self.U_device.shape[1])

    @property
    def is_sparse(self) -> bool:
        return isinstance(self.U_device, DeviceCSR)

    @property
    def dtype(self):
        return self.U_device.dtype if not self.is_sparse else self.U_device.values.dtype

    @property
    def U(self):
        if self._U_host is None:
            if self.is_sparse:
                self._U_host = self.U_device.to_scipy()
            else:
                self._U_host = self.U_device.double().cpu().numpy()
        return self._U_host

    @property
    def eta(self) -> np.ndarray:
        if self._eta_host is None:
            self._eta_host = self.eta_device.cpu().numpy()
        return self._eta_host

    def dense_u(self) -> np.ndarray:
        return self.U.toarray() if self.is_sparse else self.U

    @classmethod
    def from_host(cls, dec, dtype="float64", device=None) -> "SpectralDecomposition":
        """Upload a reference (or any duck-typed) decomposition to the device."""
        import torch

        if isinstance(dec, cls):
            return dec
        dt = N.torch_dtype(dtype)
        device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        U = dec.U
        if sp.issparse(U):
            Ud = DeviceCSR.from_scipy(sp.csr_matrix(U), dt, device)
        else:
            Ud = torch.as_tensor(np.ascontiguousarray(U, dtype=np.float64)).to(device=device, dtype=dt)
        eta = torch.as_tensor(np.asarray(dec.eta, dtype=np.float64)).to(device)
        variant = Variant(getattr(dec.variant, "value", dec.variant))
        prov = getattr(dec, "provenance", None)
        prov = Provenance(**{f: getattr(prov, f, None) for f in ("r", "p", "q", "tau", "seed")}) if prov else Provenance()
        comps = getattr(dec, "components", None) or ComponentLabeling.trivial(Ud.shape[0])
        return cls(Ud, dec.eigenvalues, eta, comps, variant, prov)


# ---------------------------------------------------------------------------
# K0: start block
# ---------------------------------------------------------------------------

def philox_key(seed: int):
    """The Philox key numpy derives for ``Philox(seed)`` (SeedSequence state)."""
    words = np.random.SeedSequence(seed & _MASK64).generate_state(2, np.uint64)
    return int(words[0]), int(words[1])


def gaussian_block(rows: int, cols: int, seed: int, row_begin: int = 0, row_end: int | None = None,
                   dtype="float64", device=None, out=None):
    """Rows [row_begin, row_end) of ``gaussian_matrix(rows, cols, seed)`` on the device."""
    import torch

    row_end = rows if row_end is None else row_end
    dt = N.torch_dtype(dtype)
    if out is None:
        out = torch.empty(row_end - row_begin, cols, dtype=dt,
                          device=device if device is not None else torch.cuda.current_device())
    ctx = N.Context.get(out.device)
    k0, k1 = philox_key(seed)
    ctx.call("gaussian_block", N.dtype_code(dt), rows, cols, row_begin, row_end, k0, k1, N.ptr(out))
    return out


def gaussian_matrix(rows: int, cols: int, seed: int, dtype="float64", device=None):
    """Standard Gaussian block from the counter-based stream (``spectral.py:55-65``), on the device."""
    return gaussian_block(rows, cols, seed, dtype=dtype, device=device)


# ---------------------------------------------------------------------------
# K3: orthonormalisation
# ---------------------------------------------------------------------------

def _gram(ctx, dt, Y, G, accumulate=False):
    n, k = Y.shape
    ctx.call("gram", dt, n, k, N.ptr(Y), Y.stride(0), N.ptr(G), int(accumulate))


def _max_dev(ctx, G) -> float:
    import ctypes

    err = ctypes.c_double()
    ctx.call("max_offdiag_error", G.shape[0], N.ptr(G), ctypes.byref(err))
    return err.value


def _trace_into(ctx, stats):
    """Append the schedule steps libfsr recorded (fsr_schedule_trace) to stats."""
    if stats is not None:
        t = ctx.lib.fsr_schedule_trace(ctx.handle)
        if t:
            stats.extend(t.decode().split(";"))


def si_flags() -> int:
    """FSR_SI_* flags of the fp32 fast-mode schedule (fsr.h fsr_si_flags), from
    the module switches SI_SPAN_ONLY / FUSED_RR / FAST_FIRST_APPLY."""
    return (1 if SI_SPAN_ONLY else 0) | (2 if FUSED_RR else 0) | (4 if FAST_FIRST_APPLY else 0)


def orthonormalize(Y, ctx=None, stats=None):
    """Replace Y by an orthonormal basis of its span (CholeskyQR2, Householder fallback).

    Mirrors ``spectral.py:165-169``: the result is checked against the
    re-orthogonalisation trigger and re-factorised when it fails.  One call of
    the operator-level ``fsr_orthonormalize`` (csrc/fsr_ops.cu): first pass on a
    7-bit Gram, second on the full Gram, Householder when Cholesky breaks down
    or max|Q^T Q - I| misses ORTH_TOL.
    """
    ctx = ctx or N.Context.get(Y.device)
    n, k = Y.shape
    ctx.call("orthonormalize", N.dtype_code(Y.dtype), n, k, N.ptr(Y), Y.stride(0))
    _trace_into(ctx, stats)
    return Y


# ---------------------------------------------------------------------------
# range finder / Rayleigh-Ritz / decompose
# ---------------------------------------------------------------------------

def _spmm(ctx, dt, Ad: DeviceCSR, X, Y):
    ctx.call("csr_spmm", dt, Ad.shape[0], N.ptr(Ad.indptr), N.ptr(Ad.indices), N.ptr(Ad.values), X.shape[1],
             N.ptr(X), X.stride(0), N.ptr(Y), Y.stride(0))


def range_finder(A, r_hat: int, q: int, seed: int, dtype="float64", device=None, stats=None,
                 _orthonormal_last: bool = True) -> RangeBasis:
    """Simultaneous iteration (``spectral.py:147-171``) on the device.

    Start block from the seeded counter stream (K0); q rounds of
    {orthonormalise (K3), B = A Q (K2)}.  Returns the last Q and B = A Q.
    One call of the operator-level ``fsr_range_finder`` (csrc/fsr_ops.cu),
    which owns the schedule: in fp32 fast mode the intermediate rounds only
    precondition (span(Q) is what reaches the output; the Gaussian start block
    already is well conditioned when r_hat <= n / 4), and with
    ``_orthonormal_last=False`` (decompose's fused path) the last basis is
    preconditioned and its exact Gram G = Q^T Q is kept for Rayleigh-Ritz.
    """
    import ctypes

    import torch

    A = SparseSymmetricMatrix.coerce(A)
    n = A.n
    if r_hat < 1 or r_hat > n:
        raise ValueError(f"r_hat must lie in [1, n], got {r_hat} for n={n}")
    if q < 1:
        raise ValueError("q must be at least 1")
    dt_t = N.torch_dtype(dtype)
    Ad = A.device(dt_t, device)
    ctx = N.Context.get(Ad.device)
    dt = N.dtype_code(dt_t)
    Q = torch.empty(n, r_hat, dtype=dt_t, device=Ad.device)
    B = torch.empty_like(Q)
    flags = si_flags() if not _orthonormal_last else si_flags() & ~2
    G = torch.empty(r_hat, r_hat, dtype=torch.float64, device=Ad.device) if flags & 2 else None
    valid = ctypes.c_int(0)
    ctx.call("range_finder", dt, n, N.ptr(Ad.indptr), N.ptr(Ad.indices), N.ptr(Ad.values), r_hat, q, seed & _MASK64,
             flags, N.ptr(Q), N.ptr(B), N.ptr(G), ctypes.byref(valid))
    _trace_into(ctx, stats)
    basis = RangeBasis(Q=Q, B=B, iterations_used=q, seed=seed)
    if valid.value:
        object.__setattr__(basis, "_gram", G)
    return basis


def _rayleigh_ritz(ctx, dt, Q, B, r, general=False):
    """C = Q^T B, eigh, U = Q V, sign fix, eta (K4-K6). Returns (U, lam, eta).

    general=True: Q is only well conditioned (decompose's fused fp32 path);
    the Ritz pairs solve C v = lambda G v with G = Q^T Q, V is G-orthonormal
    and U = Q V orthonormal -- the same pairs as orthonormalising Q first.
    One call of the operator-level ``fsr_rayleigh_ritz`` (csrc/fsr_ops.cu).
    """
    import torch

    n, k = Q.shape
    G = None
    if general is not False:
        if isinstance(general, bool):
            G = torch.empty(k, k, dtype=torch.float64, device=Q.device)
            ctx.call("gram", dt, n, k, N.ptr(Q), Q.stride(0), N.ptr(G), 0)
        else:
            G = general  # the exact Gram of Q from range_finder (fsr_rayleigh_ritz copies it)
    lam = np.empty(r, dtype=np.float64)
    U = torch.empty(n, r, dtype=Q.dtype, device=Q.device)
    eta = torch.empty(n, dtype=torch.float64, device=Q.device)
    ctx.call("rayleigh_ritz", dt, n, k, N.ptr(Q), Q.stride(0), N.ptr(B), B.stride(0), N.ptr(G), r,
             lam.ctypes.data_as(N._c_dp), N.ptr(U), U.stride(0), N.ptr(eta))
    return U, lam, eta


def approx_eigendecomposition(A, basis: RangeBasis, r: int) -> SpectralDecomposition:
    """Rayleigh-Ritz step (``spectral.py:174-198``) on the device."""
    if r < 1 or r > basis.r_hat:
        raise ValueError(f"r must lie in [1, r_hat={basis.r_hat}], got {r}")
    A = SparseSymmetricMatrix.coerce(A)
    Q, B = basis.Q, basis.B
    if Q.shape[0] != A.n:
        raise ValueError("basis dimension does not match A")
    ctx = N.Context.get(Q.device)
    # a basis from decompose's fused schedule carries its exact Gram matrix
    U, lam, eta = _rayleigh_ritz(ctx, N.dtype_code(Q.dtype), Q, B, r, general=getattr(basis, "_gram", False))
    return SpectralDecomposition(U, lam, eta, ComponentLabeling.trivial(A.n), Variant.APPROX,
                                 Provenance(r=r, p=basis.r_hat - r, q=basis.iterations_used, seed=basis.seed))


def decompose(A, r: int, p: int = DEFAULT_OVERSAMPLING, q: int = DEFAULT_POWER_ITERATIONS, seed: int = 0,
              dtype="float64", device=None) -> SpectralDecomposition:
    """Stages 1-2 (``spectral.py:297-309``): r_hat = min(r + p, n)."""
    A = SparseSymmetricMatrix.coerce(A)
    r_hat = min(r + p, A.n)
    if r > r_hat:
        raise ValueError(f"r={r} exceeds n={A.n}")
    # fp32: the last round's basis may stay merely well conditioned; the
    # Rayleigh-Ritz step then absorbs G = Q~^T Q~ (generalised eigenproblem)
    basis = range_finder(A, r_hat, q, seed, dtype=dtype, device=device,
                         _orthonormal_last=not fused_rr_enabled(dtype))
    dec = approx_eigendecomposition(A, basis, r)
    del basis
    return dec


def fused_rr_enabled(dtype) -> bool:
    """Whether decompose keeps the last SI basis non-orthonormal (fp32 fast mode)."""
    return FUSED_RR and SI_SPAN_ONLY and N.dtype_code(N.torch_dtype(dtype)) == N.F32


def mix_seed(seed: int, salt: int) -> int:
    """Decorrelated 64-bit stream seed, splitmix64 finalizer (``spectral.py:47-52``)."""
    z = (seed ^ ((salt + 1) * 0x9E3779B97F4A7C15)) & _MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK64
    return (z ^ (z >> 31)) & _MASK64


def _signfix_eta(ctx, dt, U):
    """In place: sign rule of spectral.py:133-138 on U's columns; returns eta (row norms)."""
    import torch

    n, r = U.shape
    best_abs = torch.empty(r, dtype=torch.float64, device=U.device)
    best_row = torch.empty(r, dtype=torch.int64, device=U.device)
    best_val = torch.empty(r, dtype=torch.float64, device=U.device)
    ctx.call("col_absmax", dt, n, r, N.ptr(U), U.stride(0), 0, N.ptr(best_abs), N.ptr(best_row), N.ptr(best_val))
    eta = torch.empty(n, dtype=torch.float64, device=U.device)
    ctx.call("apply_signs_rownorm", dt, n, r, N.ptr(U), U.stride(0), N.ptr(best_val), N.ptr(eta))
    return eta


def _dense_eigenpairs(A: SparseSymmetricMatrix, r: int, dtype, device=None):
    """Top-r eigenpairs of the dense A on the device (cuSOLVER syevd, fp64),
    descending with the stable order of spectral.py:141-144, sign-fixed."""
    import torch

    W = A.device(torch.float64, device)
    n = A.n
    dev = W.device
    ctx = N.Context.get(dev)
    D = torch.zeros(n, n, dtype=torch.float64, device=dev)
    if W.nnz:
        rows = torch.repeat_interleave(torch.arange(n, device=dev), W.indptr[1:] - W.indptr[:-1])
        D[rows, W.indices.long()] = W.values
    lam = np.empty(r, dtype=np.float64)
    V = torch.empty(n, r, dtype=torch.float64, device=dev)
    ctx.call("eigh_desc", n, N.ptr(D), r, lam.ctypes.data_as(N._c_dp), N.ptr(V))
    del D
    dt_t = N.torch_dtype(dtype)
    U = V if dt_t == torch.float64 else V.to(dt_t)
    eta = _signfix_eta(ctx, N.dtype_code(dt_t), U)
    return U, lam, eta


def exact_eigendecomposition(A, max_n: int = DENSE_GUARD, dtype="float64", device=None) -> SpectralDecomposition:
    """Full dense symmetric eigendecomposition (``spectral.py:200-220``), on the device."""
    A = SparseSymmetricMatrix.coerce(A)
    n = A.n
    if n > max_n:
        raise NumericalError(f"dense decomposition guarded at n <= {max_n} (got n={n}); "
                             "use the randomized path instead")
    U, lam, eta = _dense_eigenpairs(A, n, dtype, device)
    return SpectralDecomposition(U, lam, eta, ComponentLabeling.trivial(n), Variant.EXACT, Provenance(r=n))


def rank_r_decomposition(A, r: int, max_n: int = DENSE_GUARD, dtype="float64", device=None) -> SpectralDecomposition:
    """Exact decomposition truncated to the r algebraically largest pairs (``spectral.py:223-243``)."""
    A = SparseSymmetricMatrix.coerce(A)
    n = A.n
    if r < 1 or r > n:
        raise ValueError(f"r must lie in [1, n], got {r} for n={n}")
    if n > max_n:
        raise NumericalError(f"dense decomposition guarded at n <= {max_n} (got n={n}); "
                             "use the randomized path instead")
    U, lam, eta = _dense_eigenpairs(A, r, dtype, device)
    return SpectralDecomposition(U, lam, eta, ComponentLabeling.trivial(n),
                                 Variant.EXACT if r == n else Variant.RANK_R, Provenance(r=r))


def truncate_rank(dec: SpectralDecomposition, r: int) -> SpectralDecomposition:
    """Drop trailing eigenpairs (``spectral.py:246-266``)."""
    import torch

    if dec.variant is Variant.SPARSE:
        raise ValueError("cannot truncate a sparsified decomposition")
    if r < 1 or r > dec.r:
        raise ValueError(f"r must lie in [1, {dec.r}], got {r}")
    if r == dec.r:
        return dec
    U = dec.U_device[:, :r].contiguous()
    eta = torch.empty(dec.n, dtype=torch.float64, device=U.device)
    N.Context.get(U.device).call("row_norms", N.dtype_code(U.dtype), dec.n, r, N.ptr(U), U.stride(0), N.ptr(eta))
    variant = Variant.RANK_R if dec.variant is Variant.EXACT else dec.variant
    return SpectralDecomposition(U, dec.eigenvalues[:r], eta, dec.components, variant, replace(dec.provenance, r=r))


def decompose_blockwise(A, labeling: ComponentLabeling, r: int, rho: int, p: int = DEFAULT_OVERSAMPLING,
                        q: int = DEFAULT_POWER_ITERATIONS, seed: int = 0, dtype="float64",
                        device=None) -> SpectralDecomposition:
    """Per-component decomposition with a global top-r selection (``spectral.py:312-390``).

    Components of at most rho vertices are decomposed exactly (dense eigh on
    the device), larger ones by the randomized path at rank
    max(rho, ceil(r n_l / n)); the r algebraically largest pairs over all
    components are kept (ties by component, then column).  Component 0 uses
    ``seed``, later ones ``mix_seed(seed, comp)``.
    """
    import torch

    A = SparseSymmetricMatrix.coerce(A)
    n = A.n
    if labeling.n != n:
        raise ValueError("labeling does not match the matrix dimension")
    if r < 1:
        raise ValueError("r must be positive")
    if rho < 1:
        raise ValueError("rho must be positive")
    if p < 0 or q < 1:
        raise ValueError("need p >= 0 and q >= 1")
    blocks = []
    all_exact = True
    for comp in range(labeling.count):
        vertices = labeling.vertices_of(comp)
        n_l = vertices.size
        sub = A.submatrix(vertices)
        if n_l <= rho:
            part = exact_eigendecomposition(sub, max_n=max(DENSE_GUARD, n_l), dtype=dtype, device=device)
        else:
            r_l = min(max(rho, math.ceil(r * n_l / n)), n_l)
            comp_seed = seed if comp == 0 else mix_seed(seed, comp)
            part = decompose(sub, r_l, p=p, q=q, seed=comp_seed, dtype=dtype, device=device)
            all_exact = False
        blocks.append((vertices, part))

    lams = np.concatenate([part.eigenvalues for _, part in blocks])
    comps = np.concatenate([np.full(part.r, c, dtype=np.int64) for c, (_, part) in enumerate(blocks)])
    cols = np.concatenate([np.arange(part.r, dtype=np.int64) for _, part in blocks])
    order = np.lexsort((cols, comps, -lams))
    keep = order[: min(r, lams.size)]
    kept = keep.size
    dev = blocks[0][1].U_device.device
    dt_t = blocks[0][1].U_device.dtype
    U = torch.zeros(n, kept, dtype=dt_t, device=dev)
    out_cols = np.arange(kept)
    for c, (vertices, part) in enumerate(blocks):
        mine = comps[keep] == c
        if not mine.any():
            continue
        src = torch.as_tensor(cols[keep][mine], device=dev)
        dst = torch.as_tensor(out_cols[mine], device=dev)
        rows = torch.as_tensor(vertices, device=dev)
        U[rows[:, None], dst[None, :]] = part.U_device[:, src]
    eta = torch.empty(n, dtype=torch.float64, device=dev)
    N.Context.get(dev).call("row_norms", N.dtype_code(dt_t), n, kept, N.ptr(U), U.stride(0), N.ptr(eta))
    truncated = kept < lams.size
    if all_exact:
        variant = Variant.RANK_R if truncated else Variant.EXACT
    else:
        variant = Variant.APPROX
    return SpectralDecomposition(U, lams[keep], eta, labeling, variant, Provenance(r=r, p=p, q=q, seed=seed))


# ---------------------------------------------------------------------------
# K7: sparsify
# ---------------------------------------------------------------------------

HIST_BITS = 12


def key_bits(dt: int) -> int:
    return 63 if dt == N.F64 else 31


def select_threshold(hist_fn, dt: int, tau: int):
    """Radix-select the tau-th largest |u| key.

    ``hist_fn(prefix, shift, bits) -> np.uint64[2**bits]`` returns the
    (globally summed) digit histogram of nonzero keys matching ``prefix``.
    Returns (T, ties_to_take, keep): keep = min(tau, nnz) entries are the keys
    > T plus the first ``ties_to_take`` keys == T in (row, col) order.
    """
    kb = key_bits(dt)
    shift = kb - HIST_BITS
    h = hist_fn(0, shift, HIST_BITS)
    nnz = int(h.sum())
    keep = min(tau, nnz)
    if keep == nnz:
        return 0, 0, keep
    need = keep
    prefix = 0
    bits = HIST_BITS
    while True:
        cum = np.cumsum(h[::-1].astype(np.int64))
        pos = int(np.searchsorted(cum, need))  # first bin (from the top) reaching need
        b = (1 << bits) - 1 - pos
        above = int(cum[pos] - h[b])
        need -= above
        prefix |= b << shift
        if shift == 0:
            return prefix, need, keep
        bits = min(HIST_BITS, shift)
        shift -= bits
        h = hist_fn(prefix, shift, bits)


def sparsify(dec: SpectralDecomposition, tau: int) -> SpectralDecomposition:
    """Keep the tau largest-magnitude entries of U, ties in (row, col) order
    (``spectral.py:269-294``); eta is recomputed from the kept U."""
    import torch

    if not isinstance(dec, SpectralDecomposition):
        dec = SpectralDecomposition.from_host(dec)
    if dec.variant is Variant.SPARSE:
        raise ValueError("decomposition is already sparse")
    if tau < 1:
        raise ValueError("tau must be positive")
    import ctypes

    U = dec.U_device
    n, r = U.shape
    ctx = N.Context.get(U.device)
    dt = N.dtype_code(U.dtype)
    # operator level (csrc/fsr_ops.cu): radix-select the tau-th |u| key, then compact
    T, ties, keep = ctypes.c_uint64(), ctypes.c_int64(), ctypes.c_int64()
    ctx.call("sparsify_select", dt, n, r, N.ptr(U), U.stride(0), tau, ctypes.byref(T), ctypes.byref(ties),
             ctypes.byref(keep))
    cap = max(1, int(keep.value))
    indptr = torch.empty(n + 1, dtype=torch.int64, device=U.device)
    indices = torch.empty(cap, dtype=torch.int32, device=U.device)
    values = torch.empty(cap, dtype=U.dtype, device=U.device)
    eta = torch.empty(n, dtype=torch.float64, device=U.device)
    nnz = ctypes.c_int64()
    ctx.call("sparsify_apply", dt, n, r, N.ptr(U), U.stride(0), T.value, ties.value, N.ptr(indptr), N.ptr(indices),
             N.ptr(values), N.ptr(eta), ctypes.byref(nnz))
    k = int(nnz.value)
    Ut = DeviceCSR(indptr, indices[:k], values[:k], (n, r))
    return SpectralDecomposition(Ut, dec.eigenvalues, eta, dec.components, Variant.SPARSE,
                                 replace(dec.provenance, tau=tau))


def compact_rows(ctx, dt, U, T, tie_offset, ties_to_take, capacity, counts=None):
    """Count + compact the kept entries of the local rows of U into a DeviceCSR."""
    import ctypes

    import torch

    n, r = U.shape
    if counts is None:
        gt = torch.empty(n, dtype=torch.int64, device=U.device)
        eq = torch.empty(n, dtype=torch.int64, device=U.device)
        ctx.call("threshold_counts", dt, n, r, N.ptr(U), U.stride(0), T, N.ptr(gt), N.ptr(eq))
    else:
        gt, eq = counts
    indptr = torch.empty(n + 1, dtype=torch.int64, device=U.device)
    cap = max(1, int(capacity))
    indices = torch.empty(cap, dtype=torch.int32, device=U.device)
    values = torch.empty(cap, dtype=U.dtype, device=U.device)
    eta = torch.empty(n, dtype=torch.float64, device=U.device)
    nnz = ctypes.c_int64()
    ctx.call("threshold_compact", dt, n, r, N.ptr(U), U.stride(0), T, tie_offset, ties_to_take, N.ptr(gt),
             N.ptr(eq), N.ptr(indptr), N.ptr(indices), N.ptr(values), N.ptr(eta), ctypes.byref(nnz))
    k = int(nnz.value)
    return DeviceCSR(indptr, indices[:k], values[:k], (n, r)), eta


def row_norms(U) -> np.ndarray:
    """Host helper matching ``spectral.py:127-130``."""
    if sp.issparse(U):
        return np.sqrt(np.asarray(U.multiply(U).sum(axis=1)).ravel())
    return np.linalg.norm(U, axis=1)
