"""Numpy implementation of the sharded path's local ops (TEST INFRASTRUCTURE).

Lets tests drive paper_1703_06935_b200.distributed's orchestration (which
collectives, in which order, with which offsets) on CPU with the gloo
backend; the arithmetic follows the oracle (float64).
"""

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp
import torch

from oracle import fsr_oracle as O


def _np(t):
    return t.numpy() if isinstance(t, torch.Tensor) else t


def _t(a):
    return torch.as_tensor(np.ascontiguousarray(a))


class NumpyOps:
    def gaussian(self, n, cols, seed, r0, r1):
        return _t(O.gaussian_matrix(n, cols, seed)[r0:r1])

    def spmm(self, A_local, X_full):
        return _t(A_local @ _np(X_full))

    def spmm_into(self, A_local, X, Y):
        Y.copy_(_t(A_local @ _np(X)))
        return Y

    def empty(self, rows, cols):
        return torch.empty(rows, cols, dtype=torch.float64)

    def gram(self, Y, fast=False):
        y = _np(Y)
        return _t(y.T @ y)

    def max_dev(self, G):
        g = _np(G)
        return float(np.abs(g - np.eye(g.shape[0])).max())

    def cholesky(self, G):
        try:
            return _t(np.linalg.cholesky(_np(G)).T)
        except np.linalg.LinAlgError:
            return None

    def apply_rinv(self, R, Y, fast=False):
        return _t(sla.solve_triangular(_np(R), _np(Y).T, trans="T", lower=False).T)

    def householder(self, Yfull):
        return _t(np.linalg.qr(_np(Yfull))[0])

    def cross(self, Q, B):
        return _t(_np(Q).T @ _np(B))

    def eigh_desc(self, C, r):
        c = _np(C)
        lam, V = np.linalg.eigh((c + c.T) / 2.0)
        pick = np.argsort(-lam, kind="stable")[:r]
        return lam[pick], _t(V[:, pick])

    def lift(self, Q, V):
        return _t(_np(Q) @ _np(V))

    def col_absmax(self, U, row_offset):
        u = _np(U)
        if u.shape[0] == 0:
            r = u.shape[1]
            return _t(np.full(r, -1.0)), _t(np.full(r, np.iinfo(np.int64).max)), _t(np.zeros(r))
        lead = np.argmax(np.abs(u), axis=0)
        cols = np.arange(u.shape[1])
        return _t(np.abs(u[lead, cols])), _t((lead + row_offset).astype(np.int64)), _t(u[lead, cols])

    def apply_signs(self, U, best_val):
        s = np.sign(_np(best_val))
        s[s == 0] = 1.0
        u = _np(U)
        u *= s
        return _t(np.linalg.norm(u, axis=1))

    @staticmethod
    def _keys(u):
        return np.abs(u).view(np.uint64) & np.uint64(0x7FFFFFFFFFFFFFFF)

    def histogram(self, U, prefix, shift, bits):
        k = self._keys(_np(U)).ravel()
        hi = 0 if shift + bits >= 64 else (~((1 << (shift + bits)) - 1)) & ((1 << 64) - 1)
        sel = (k != 0) & ((k & np.uint64(hi)) == np.uint64(prefix & hi))
        d = ((k[sel] >> np.uint64(shift)) & np.uint64((1 << bits) - 1)).astype(np.int64)
        return _t(np.bincount(d, minlength=1 << bits).astype(np.int64))

    def counts(self, U, T):
        k = self._keys(_np(U))
        T = np.uint64(T)
        return _t((k > T).sum(axis=1).astype(np.int64)), _t(((k == T) & (k != 0)).sum(axis=1).astype(np.int64))

    def compact(self, U, T, tie_offset, ties, gt, eq):
        u = _np(U)
        k = self._keys(u)
        T = np.uint64(T)
        rows, cols, vals = [], [], []
        tie = tie_offset
        for i in range(u.shape[0]):
            for j in range(u.shape[1]):
                take = k[i, j] > T
                if k[i, j] == T and k[i, j] != 0:
                    take = tie < ties
                    tie += 1
                if take:
                    rows.append(i)
                    cols.append(j)
                    vals.append(u[i, j])
        M = sp.csr_matrix((vals, (rows, cols)), shape=u.shape)
        M.sort_indices()
        return M, np.sqrt(np.asarray(M.multiply(M).sum(axis=1)).ravel())
