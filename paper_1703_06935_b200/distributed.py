"""Row-sharded offline FSR across GPUs (one process per GPU).

Partitioning: contiguous row blocks of W, the start block,
Q, B and U, balanced by nonzeros.  Per simultaneous-iteration round:

  * orthonormalise the local rows: the Gram partials B_l^T B_l are summed
    across ranks (fp64, in rank order -> bitwise identical on every rank),
    every rank factors the same r_hat x r_hat Gram redundantly and applies
    R^-1 to its own rows (CholeskyQR2; Householder on the gathered block as
    the rank-deficient fallback, spectral.py:165-169);
  * all-gather the Q row shards, then B_l = W_l Q locally (the exchange step).

Rayleigh-Ritz: C = sum_l Q_l^T B_l (rank-ordered), redundant eigh, local
U_l = Q_l V, column signs from the all-gathered per-rank (|u|max, row, u).
Thresholding: digit histograms summed across ranks, per-rank tie counts
all-gathered so every rank knows how many ties lower ranks hold (the global
(row, col) tie order is rank order then local order), local compaction.

Collectives go through ``Comm`` (torch.distributed; NCCL on GPUs, gloo in the
CPU tests); local arithmetic through an ops object (``CudaOps`` = libfsr;
tests inject a numpy implementation to check the orchestration on CPU).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N
from .spectral import HIST_BITS, ORTH_TOL, key_bits, select_threshold


# ---------------------------------------------------------------------------
# communication
# ---------------------------------------------------------------------------

class Comm:
    """Thin wrapper over torch.distributed with deterministic reductions."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.backend = dist.get_backend(group) if dist.is_initialized() else "none"

    def _staged(self, t):
        # gloo has no CUDA collectives for everything we need: stage through host memory
        if self.backend == "gloo" and t.is_cuda:
            return t.cpu(), t.device
        return t, None

    def all_gather(self, t):
        """List of every rank's tensor (same shape on every rank)."""
        import torch

        if self.world == 1:
            return [t]
        src, dev = self._staged(t.contiguous())
        out = [torch.empty_like(src) for _ in range(self.world)]
        self.dist.all_gather(out, src, group=self.group)
        return [o.to(dev) for o in out] if dev is not None else out

    def all_gather_rows(self, t, counts, out=None, async_op=False):
        """Concatenate row shards of different lengths (counts[r] rows on rank r)
        straight into ``out`` (allocated when None): one broadcast per rank into
        its row range of the output -- no padding, no concatenation copy.  With
        ``async_op`` returns (out, handle); ``handle.wait()`` orders the current
        stream after the transfer."""
        import torch

        if self.world == 1:
            if out is None:
                return (t, _Done()) if async_op else t
            out.copy_(t)
            return (out, _Done()) if async_op else out
        rows = int(sum(counts))
        if out is None:
            out = torch.empty((rows,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        staged = self.backend == "gloo" and out.is_cuda
        buf = out.cpu() if staged else out
        src = t.cpu() if staged and t.is_cuda else t
        offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
        if len(set(counts)) == 1 and not staged:
            work = [self.dist.all_gather_into_tensor(buf, src.contiguous(), group=self.group, async_op=True)]
        else:
            me = buf[int(offs[self.rank]):int(offs[self.rank + 1])]
            me.copy_(src)
            work = [self.dist.broadcast(buf[int(offs[r]):int(offs[r + 1])], src=self._global(r), group=self.group,
                                        async_op=True) for r in range(self.world) if counts[r] > 0]
        handle = _Handles(work, (lambda: out.copy_(buf)) if staged else None)
        if async_op:
            return out, handle
        handle.wait()
        return out

    def _global(self, r):
        return r if self.group is None else self.dist.get_global_rank(self.group, r)

    def sum_ordered(self, t):
        """Sum over ranks in rank order, bitwise identical on every rank.

        Reduce-scatter by hand so the order is fixed: the flattened tensor is
        cut into world equal chunks, an all-to-all hands chunk c of every
        rank's partial to rank c, which adds them in rank order
        (((p_0 + p_1) + p_2) + ...); an all-gather returns the reduced
        chunks.  Peak extra memory is ~2 copies of t per rank (the old
        all-gather of every partial needed world copies: 7.7 GB per r_hat^2
        fp64 Gram at C4 on 8 ranks)."""
        import torch

        if self.world == 1:
            return t
        src, dev = self._staged(t.contiguous())
        flat = src.reshape(-1)
        m = -(-flat.numel() // self.world)
        send = torch.zeros(m * self.world, dtype=flat.dtype, device=flat.device)
        send[:flat.numel()] = flat
        recv = torch.empty_like(send)
        self.dist.all_to_all_single(recv, send, group=self.group)
        del send
        parts = recv.view(self.world, m)
        mine = parts[0].clone()
        for k in range(1, self.world):
            mine += parts[k]
        del recv, parts
        full = torch.empty(m * self.world, dtype=flat.dtype, device=flat.device)
        self.dist.all_gather_into_tensor(full, mine, group=self.group)
        res = full[:flat.numel()].view(t.shape)
        return res.to(dev) if dev is not None else res

    def barrier(self):
        if self.world > 1:
            self.dist.barrier(group=self.group)


class _Done:
    def wait(self):
        return None


class _Handles:
    """Several async collectives (+ an optional host->device copy back) as one handle."""

    def __init__(self, work, finish=None):
        self.work, self.finish = work, finish

    def wait(self):
        for w in self.work:
            w.wait()
        if self.finish is not None:
            self.finish()
            self.finish = None


# ---------------------------------------------------------------------------
# partitioning
# ---------------------------------------------------------------------------

def row_partition(indptr: np.ndarray, world: int):
    """Contiguous row blocks with ~equal nonzeros (empty blocks allowed)."""
    indptr = np.asarray(indptr, dtype=np.int64)
    n = indptr.size - 1
    nnz = int(indptr[-1])
    cuts = [0]
    for r in range(1, world):
        c = int(np.searchsorted(indptr, (nnz * r) // world, side="left")) if nnz else (n * r) // world
        cuts.append(min(max(c, cuts[-1]), n))
    cuts.append(n)
    return [(cuts[i], cuts[i + 1]) for i in range(world)]


@dataclass
class Shard:
    rank: int
    world: int
    n: int
    r0: int
    r1: int
    counts: list

    @property
    def rows(self) -> int:
        return self.r1 - self.r0


def make_shard(comm: Comm, indptr: np.ndarray) -> Shard:
    parts = row_partition(indptr, comm.world)
    r0, r1 = parts[comm.rank]
    return Shard(comm.rank, comm.world, int(len(indptr) - 1), r0, r1, [b - a for a, b in parts])


# ---------------------------------------------------------------------------
# local ops on the device
# ---------------------------------------------------------------------------

class CudaOps:
    """Local arithmetic of the sharded path through libfsr."""

    def __init__(self, device, dtype="float32"):
        import torch

        self.torch = torch
        self.device = torch.device(device)
        self.dt_t = N.torch_dtype(dtype)
        self.dt = N.dtype_code(self.dt_t)
        self.ctx = N.Context.get(self.device)

    def gaussian(self, n, cols, seed, r0, r1):
        from .spectral import gaussian_block

        return gaussian_block(n, cols, seed, r0, r1, dtype=self.dt_t, device=self.device)

    def spmm(self, A_local, X_full):
        Y = self.torch.empty(A_local.shape[0], X_full.shape[1], dtype=self.dt_t, device=self.device)
        return self.spmm_into(A_local, X_full, Y)

    def spmm_into(self, A_local, X, Y):
        """Y = A_local X for a column panel (Y may be a column slice of a wider block)."""
        self.ctx.call("csr_spmm", self.dt, A_local.shape[0], N.ptr(A_local.indptr), N.ptr(A_local.indices),
                      N.ptr(A_local.values), X.shape[1], N.ptr(X), X.stride(0), N.ptr(Y), Y.stride(0))
        return Y

    def empty(self, rows, cols):
        return self.torch.empty(rows, cols, dtype=self.dt_t, device=self.device)

    def gram(self, Y, fast=False):
        k = Y.shape[1]
        G = self.torch.empty(k, k, dtype=self.torch.float64, device=self.device)
        if fast and self.dt == N.F32:  # first CholeskyQR pass: one-slice Gram (spectral._cholqr_pass)
            self.ctx.call("gram_levels", Y.shape[0], k, N.ptr(Y), Y.stride(0), N.ptr(G), 0, 1)
        else:
            self.ctx.call("gram", self.dt, Y.shape[0], k, N.ptr(Y), Y.stride(0), N.ptr(G), 0)
        return G

    def max_dev(self, G) -> float:
        import ctypes

        err = ctypes.c_double()
        self.ctx.call("max_offdiag_error", G.shape[0], N.ptr(G), ctypes.byref(err))
        return err.value

    def cholesky(self, G):
        R = G.clone()
        st = self.ctx.call("cholesky", R.shape[0], N.ptr(R))
        return None if st == N.ENOTSPD else R

    def apply_rinv(self, R, Y, fast=False):
        # first CholeskyQR pass: R^-1 may enter as a 7-bit matrix (spectral._cholqr_pass)
        from .spectral import FAST_FIRST_APPLY

        self.ctx.call("apply_rinv_levels", self.dt, Y.shape[0], Y.shape[1], N.ptr(R), N.ptr(Y), Y.stride(0),
                      1 if (fast and FAST_FIRST_APPLY) else 4)
        return Y

    def householder(self, Yfull):
        self.ctx.call("householder_qr", self.dt, Yfull.shape[0], Yfull.shape[1], N.ptr(Yfull), Yfull.stride(0))
        return Yfull

    def cross(self, Q, B):
        k = Q.shape[1]
        C = self.torch.empty(k, k, dtype=self.torch.float64, device=self.device)
        self.ctx.call("cross", self.dt, Q.shape[0], k, N.ptr(Q), Q.stride(0), N.ptr(B), B.stride(0), N.ptr(C), 0)
        return C

    def eigh_desc(self, C, r):
        lam = np.empty(r, dtype=np.float64)
        V = self.torch.empty(C.shape[0], r, dtype=self.torch.float64, device=self.device)
        Cw = C.clone()
        self.ctx.call("eigh_desc", C.shape[0], N.ptr(Cw), r, lam.ctypes.data_as(N._c_dp), N.ptr(V))
        return lam, V

    def lift(self, Q, V):
        r = V.shape[1]
        U = self.torch.empty(Q.shape[0], r, dtype=self.dt_t, device=self.device)
        self.ctx.call("lift", self.dt, Q.shape[0], Q.shape[1], r, N.ptr(Q), Q.stride(0), N.ptr(V), N.ptr(U),
                      U.stride(0))
        return U

    def col_absmax(self, U, row_offset):
        r = U.shape[1]
        t = self.torch
        a = t.empty(r, dtype=t.float64, device=self.device)
        row = t.empty(r, dtype=t.int64, device=self.device)
        v = t.empty(r, dtype=t.float64, device=self.device)
        self.ctx.call("col_absmax", self.dt, U.shape[0], r, N.ptr(U), U.stride(0), row_offset, N.ptr(a), N.ptr(row),
                      N.ptr(v))
        return a, row, v

    def apply_signs(self, U, best_val):
        eta = self.torch.empty(U.shape[0], dtype=self.torch.float64, device=self.device)
        self.ctx.call("apply_signs_rownorm", self.dt, U.shape[0], U.shape[1], N.ptr(U), U.stride(0), N.ptr(best_val),
                      N.ptr(eta))
        return eta

    def histogram(self, U, prefix, shift, bits):
        h = self.torch.zeros(1 << bits, dtype=self.torch.int64, device=self.device)
        self.ctx.call("abs_histogram", self.dt, U.shape[0], U.shape[1], N.ptr(U), U.stride(0), prefix, shift, bits,
                      N.ptr(h))
        return h

    def counts(self, U, T):
        t = self.torch
        gt = t.empty(U.shape[0], dtype=t.int64, device=self.device)
        eq = t.empty(U.shape[0], dtype=t.int64, device=self.device)
        self.ctx.call("threshold_counts", self.dt, U.shape[0], U.shape[1], N.ptr(U), U.stride(0), T, N.ptr(gt),
                      N.ptr(eq))
        return gt, eq

    def compact(self, U, T, tie_offset, ties, gt, eq):
        from .spectral import compact_rows

        capacity = int(gt.sum().item()) + int(eq.sum().item())
        return compact_rows(self.ctx, self.dt, U, T, tie_offset, ties, capacity, counts=(gt, eq))


# ---------------------------------------------------------------------------
# the sharded algorithm
# ---------------------------------------------------------------------------

def sharded_orthonormalize(comm: Comm, ops, Y, shard: Shard, dt_code: int, stats=None):
    """CholeskyQR2 over row shards; Householder on the gathered block as fallback."""
    ok = True
    last_dev = np.inf
    for pass_ in range(2):
        G = comm.sum_ordered(ops.gram(Y, fast=(pass_ == 0)))
        last_dev = ops.max_dev(G)
        R = ops.cholesky(G)
        if R is None:
            ok = False
            break
        Y = ops.apply_rinv(R, Y, fast=(pass_ == 0))
    method = "cholqr2"
    if ok and last_dev > 0.1:
        G = comm.sum_ordered(ops.gram(Y))
        ok = ops.max_dev(G) <= ORTH_TOL[dt_code]
        method = "cholqr2+check"
    if not ok:
        full = comm.all_gather_rows(Y, shard.counts)
        full = ops.householder(full.contiguous())
        Y = full[shard.r0:shard.r1].contiguous()
        method = "householder"
    if stats is not None:
        stats.append(method)
    return Y


def sharded_range_finder(comm: Comm, ops, A_local, shard: Shard, r_hat: int, q: int, seed: int, dt_code: int,
                         stats=None):
    """Q, B row shards of spectral.range_finder (spectral.py:147-171)."""
    if r_hat < 1 or r_hat > shard.n:
        raise ValueError(f"r_hat must lie in [1, n], got {r_hat} for n={shard.n}")
    if q < 1:
        raise ValueError("q must be at least 1")
    from .spectral import SI_SPAN_ONLY

    Y = ops.gaussian(shard.n, r_hat, seed, shard.r0, shard.r1)
    Q = None
    for t in range(q):
        if SI_SPAN_ONLY and dt_code == N.F32 and t < q - 1:
            # intermediate rounds: a well-conditioned basis suffices (spectral.range_finder)
            Q = Y if (t == 0 and 4 * r_hat <= shard.n) else sharded_precondition(comm, ops, Y, shard, dt_code, stats)
        else:
            Q = sharded_orthonormalize(comm, ops, Y, shard, dt_code, stats)
        Y = exchange_spmm(comm, ops, A_local, Q, shard)
    return Q, Y


# Column-panel width of the pipelined exchange (EXCHANGE_PANEL columns of all n
# rows per buffer, two buffers): at C4 (n = 2.5e6, fp32) 2 x 5.1 GB instead of
# the 110 GB gathered block.  0 = gather the whole block at once.
EXCHANGE_PANEL = 512


def exchange_spmm(comm: Comm, ops, A_local, Q, shard: Shard, panel: int | None = None):
    """B_l = W_l Q (the SI exchange step, spectral.py:170) without holding all of Q.

    Q's columns are exchanged in panels: panel j+1's all-gather (one broadcast
    per rank into its row range of a preallocated n x w buffer) is in flight
    while K2 multiplies panel j into B_l[:, panel j]; two panel buffers
    alternate.  K2 sums each row's nonzeros in the same order whatever the
    panel width, so B_l is bitwise the unpipelined product.  Per-rank memory:
    Q_l + B_l + 2 n w."""
    w_all = Q.shape[1]
    panel = EXCHANGE_PANEL if panel is None else panel
    if comm.world == 1 or panel <= 0 or panel >= w_all:
        return ops.spmm(A_local, comm.all_gather_rows(Q, shard.counts))
    B = ops.empty(shard.rows, w_all)
    bufs = [ops.empty(shard.n * panel, 1), ops.empty(shard.n * panel, 1)]
    npan = -(-w_all // panel)

    def start(j):
        c0, c1 = j * panel, min(w_all, (j + 1) * panel)
        out = bufs[j % 2][: shard.n * (c1 - c0)].view(shard.n, c1 - c0)
        return comm.all_gather_rows(Q[:, c0:c1].contiguous(), shard.counts, out=out, async_op=True)

    cur = start(0)
    for j in range(npan):
        panel_j, handle = cur
        handle.wait()
        if j + 1 < npan:
            cur = start(j + 1)  # in flight while K2 runs on panel j
        c0, c1 = j * panel, min(w_all, (j + 1) * panel)
        ops.spmm_into(A_local, panel_j, B[:, c0:c1])
    return B


def sharded_precondition(comm: Comm, ops, Y, shard: Shard, dt_code: int, stats=None):
    """spectral._precondition over row shards: one 7-bit CholeskyQR pass, a 7-bit
    Gram check, full CholeskyQR2 if the basis is not within PRECOND_TOL of orthonormal."""
    from .spectral import PRECOND_TOL

    R = ops.cholesky(comm.sum_ordered(ops.gram(Y, fast=True)))
    if R is not None:
        Y1 = ops.apply_rinv(R, Y, fast=True)
        if ops.max_dev(comm.sum_ordered(ops.gram(Y1, fast=True))) <= PRECOND_TOL:
            if stats is not None:
                stats.append("precond")
            return Y1
        Y = Y1
    return sharded_orthonormalize(comm, ops, Y, shard, dt_code, stats)


def sharded_rayleigh_ritz(comm: Comm, ops, Q, B, r: int, shard: Shard):
    """Local U rows, eigenvalues and eta of spectral.approx_eigendecomposition."""
    import torch

    C = comm.sum_ordered(ops.cross(Q, B))
    lam, V = ops.eigh_desc(C, r)
    U = ops.lift(Q, V)
    a, row, v = ops.col_absmax(U, shard.r0)
    A = comm.all_gather(a)
    Rw = comm.all_gather(row)
    Vv = comm.all_gather(v)
    best_a, best_row, best_v = A[0].clone(), Rw[0].clone(), Vv[0].clone()
    for pa, pr, pv in zip(A[1:], Rw[1:], Vv[1:]):
        better = (pa > best_a) | ((pa == best_a) & (pr < best_row))
        best_a = torch.where(better, pa, best_a)
        best_row = torch.where(better, pr, best_row)
        best_v = torch.where(better, pv, best_v)
    eta = ops.apply_signs(U, best_v)
    return U, lam, eta


def sharded_sparsify(comm: Comm, ops, U, tau: int, shard: Shard, dt_code: int):
    """Local CSR rows of spectral.sparsify (spectral.py:269-294) with a global tau."""
    import torch

    def hist_fn(prefix, shift, bits):
        h = comm.sum_ordered(ops.histogram(U, prefix, shift, bits))
        return h.cpu().numpy().astype(np.uint64)

    T, ties, keep = select_threshold(hist_fn, dt_code, tau)
    gt, eq = ops.counts(U, T)
    eq_local = torch.tensor([int(eq.sum().item())], dtype=torch.int64, device=eq.device)
    eq_all = [int(x.item()) for x in comm.all_gather(eq_local)]
    tie_offset = sum(eq_all[: shard.rank])
    Ut, eta = ops.compact(U, T, tie_offset, ties, gt, eq)
    return Ut, eta, keep


__all__ = ["Comm", "CudaOps", "Shard", "make_shard", "row_partition", "sharded_orthonormalize",
           "sharded_range_finder", "sharded_rayleigh_ritz", "sharded_sparsify", "exchange_spmm", "HIST_BITS",
           "key_bits"]


def shard_rows(A, r0: int, r1: int):
    """Rows [r0, r1) of a DeviceCSR (global column indices kept)."""
    from .sparsemat import DeviceCSR

    ip = A.indptr[r0:r1 + 1]
    e0, e1 = int(ip[0].item()), int(ip[-1].item())
    return DeviceCSR((ip - e0).contiguous(), A.indices[e0:e1], A.values[e0:e1], (r1 - r0, A.shape[1]))


def gather_csr(comm: Comm, local, shard: Shard):
    """Replicate a row-sharded DeviceCSR on every rank (for the online replicas)."""
    import torch

    from .sparsemat import DeviceCSR

    nnz = torch.tensor([local.nnz], dtype=torch.int64, device=local.values.device)
    nnzs = [int(x.item()) for x in comm.all_gather(nnz)]
    indices = comm.all_gather_rows(local.indices.unsqueeze(1), nnzs).squeeze(1)
    values = comm.all_gather_rows(local.values.unsqueeze(1), nnzs).squeeze(1)
    ptr_parts = comm.all_gather_rows(local.indptr[1:].unsqueeze(1), shard.counts).squeeze(1)
    offsets = np.concatenate([[0], np.cumsum(nnzs)])
    # add each rank's nnz offset to its row pointers
    add = torch.repeat_interleave(torch.as_tensor(offsets[:-1], device=ptr_parts.device),
                                  torch.as_tensor(shard.counts, device=ptr_parts.device))
    indptr = torch.cat([torch.zeros(1, dtype=torch.int64, device=ptr_parts.device), ptr_parts + add])
    return DeviceCSR(indptr, indices.contiguous(), values.contiguous(), (shard.n, local.shape[1]))


def sharded_decompose(comm: Comm, S, r: int, p: int, q: int, seed: int = 0, tau: int | None = None,
                      dtype="float32", device=None, stats=None):
    """End-to-end sharded offline pipeline on GPUs.  Returns a local-rows result
    dict (Q/B freed): U rows, eigenvalues, eta rows and, with tau, the local
    sparse rows."""
    import torch

    from .sparsemat import SparseSymmetricMatrix

    S = SparseSymmetricMatrix.coerce(S)
    device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    ops = CudaOps(device, dtype)
    A = S.device(ops.dt_t, device)
    shard = make_shard(comm, A.indptr.cpu().numpy())
    A_local = shard_rows(A, shard.r0, shard.r1)
    r_hat = min(r + p, shard.n)
    Q, B = sharded_range_finder(comm, ops, A_local, shard, r_hat, q, seed, ops.dt, stats)
    U, lam, eta = sharded_rayleigh_ritz(comm, ops, Q, B, r, shard)
    del Q, B
    out = {"shard": shard, "U": U, "eigenvalues": lam, "eta": eta}
    if tau is not None:
        Ut, eta_s, keep = sharded_sparsify(comm, ops, U, tau, shard, ops.dt)
        out.update(Ut=Ut, eta_sparse=eta_s, kept=keep)
    return out
