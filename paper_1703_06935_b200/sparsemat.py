"""Symmetric CSR operator on the host and/or the device.

Mirrors the reference ``SparseSymmetricMatrix`` (``sparsemat.py:19-86``):
the same constructor validation (square, symmetric within 1e-12) and
canonicalisation (``from_scipy``: float64, duplicates summed, zeros
eliminated, sorted indices).  On top of that the matrix can live on a CUDA
device (``DeviceCSR``: int64 row pointers, int32 columns, fp32/fp64 values),
which is what the kernels consume; the host copy is materialised lazily.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp

SYMMETRY_TOL = 1e-12


class DeviceCSR:
    """CSR block on a CUDA device: rows x cols, int64 indptr, int32 indices."""

    def __init__(self, indptr, indices, values, shape):
        self.indptr = indptr
        self.indices = indices
        self.values = values
        self.shape = (int(shape[0]), int(shape[1]))

    @property
    def nnz(self) -> int:
        return int(self.indices.numel())

    @property
    def dtype(self):
        return self.values.dtype

    @property
    def device(self):
        return self.values.device

    @classmethod
    def from_scipy(cls, csr, dtype, device) -> "DeviceCSR":
        import torch

        csr = sp.csr_matrix(csr)
        return cls(
            torch.as_tensor(csr.indptr.astype(np.int64)).to(device),
            torch.as_tensor(csr.indices.astype(np.int32)).to(device),
            torch.as_tensor(np.asarray(csr.data, dtype=np.float64)).to(device=device, dtype=dtype),
            csr.shape,
        )

    def to_scipy(self) -> sp.csr_matrix:
        return sp.csr_matrix(
            (self.values.double().cpu().numpy(), self.indices.cpu().numpy(), self.indptr.cpu().numpy()),
            shape=self.shape,
        )

    def astype(self, dtype) -> "DeviceCSR":
        if dtype == self.values.dtype:
            return self
        return DeviceCSR(self.indptr, self.indices, self.values.to(dtype), self.shape)


def _validate(mat) -> None:
    if not sp.issparse(mat):
        raise ValueError("csr must be a scipy sparse matrix")
    if mat.shape[0] != mat.shape[1]:
        raise ValueError(f"matrix must be square, got shape {mat.shape}")
    if mat.nnz:
        asym = abs(mat - mat.T)
        if asym.nnz and asym.max() > SYMMETRY_TOL:
            raise ValueError(f"matrix is not symmetric within {SYMMETRY_TOL:g} (max deviation {asym.max():.3g})")


class SparseSymmetricMatrix:
    """Square matrix with entry (i, j) equal to (j, i) within 1e-12.

    Construct from a scipy matrix (validated like the reference) or, for
    device-built graphs, with ``from_device`` (symmetric by construction; the
    O(nnz) host check is skipped because no host copy exists).
    """

    def __init__(self, csr=None, *, device_csr: DeviceCSR | None = None, validate: bool = True):
        if csr is None and device_csr is None:
            raise ValueError("need a host or a device matrix")
        if csr is not None and validate:
            _validate(csr)
        self._csr = csr
        self._dev = {}
        if device_csr is not None:
            self._dev[(device_csr.values.dtype, device_csr.device)] = device_csr
            self._shape = device_csr.shape
            self._nnz = device_csr.nnz
        else:
            self._shape = csr.shape
            self._nnz = csr.nnz

    # -- constructors mirroring sparsemat.py:39-53 --------------------------
    @classmethod
    def from_scipy(cls, mat) -> "SparseSymmetricMatrix":
        csr = sp.csr_matrix(mat, dtype=np.float64, copy=True)
        csr.sum_duplicates()
        csr.eliminate_zeros()
        csr.sort_indices()
        return cls(csr)

    @classmethod
    def from_dense(cls, arr) -> "SparseSymmetricMatrix":
        return cls.from_scipy(np.asarray(arr, dtype=np.float64))

    @classmethod
    def identity(cls, n: int) -> "SparseSymmetricMatrix":
        return cls(sp.identity(n, dtype=np.float64, format="csr"))

    @classmethod
    def from_device(cls, device_csr: DeviceCSR) -> "SparseSymmetricMatrix":
        return cls(device_csr=device_csr)

    @classmethod
    def coerce(cls, A) -> "SparseSymmetricMatrix":
        """Accept this class, the reference's (duck-typed ``.csr``), scipy, or DeviceCSR."""
        if isinstance(A, cls):
            return A
        if isinstance(A, DeviceCSR):
            return cls.from_device(A)
        if hasattr(A, "csr") and sp.issparse(A.csr):
            return cls(sp.csr_matrix(A.csr), validate=False)  # the reference validated it already
        if sp.issparse(A):
            return cls.from_scipy(A)
        raise ValueError(f"cannot interpret {type(A).__name__} as a symmetric sparse matrix")

    # -- properties ----------------------------------------------------------
    @property
    def csr(self) -> sp.csr_matrix:
        if self._csr is None:
            dev = next(iter(self._dev.values()))
            self._csr = dev.to_scipy()
        return self._csr

    @property
    def shape(self):
        return self._shape

    @property
    def n(self) -> int:
        return self._shape[0]

    @property
    def nnz(self) -> int:
        return self._nnz

    def device(self, dtype, device=None) -> DeviceCSR:
        """The matrix on ``device`` with values in ``dtype`` (cached)."""
        import torch

        device = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
        if device.index is None:
            device = torch.device("cuda", torch.cuda.current_device())
        key = (dtype, device)
        if key not in self._dev:
            src = next((d for (dt, dv), d in self._dev.items() if dv == device), None)
            if src is not None:
                self._dev[key] = src.astype(dtype)
            else:
                self._dev[key] = DeviceCSR.from_scipy(self.csr, dtype, device)
        return self._dev[key]

    def __matmul__(self, other):
        return self.csr @ other

    def matvec(self, x):
        return self.csr @ np.asarray(x)

    def to_dense(self) -> np.ndarray:
        return self.csr.toarray()

    def diagonal(self) -> np.ndarray:
        return self.csr.diagonal()

    def submatrix(self, index) -> "SparseSymmetricMatrix":
        """Principal submatrix on the given sorted vertex indices (``sparsemat.py:82-86``),
        extracted on the device (fp64 values); canonical CSR, device-resident."""
        import torch

        W = self.device(torch.float64)
        dev = W.device
        idx = torch.as_tensor(np.asarray(index, dtype=np.int64)).to(dev)
        m = int(idx.numel())
        newid = torch.full((self.n,), -1, dtype=torch.int64, device=dev)
        newid[idx] = torch.arange(m, device=dev)
        starts = W.indptr[idx]
        lens = W.indptr[idx + 1] - starts
        total = int(lens.sum())
        rows = torch.repeat_interleave(torch.arange(m, device=dev), lens)
        first = torch.cumsum(lens, 0) - lens
        pos = torch.repeat_interleave(starts - first, lens) + torch.arange(total, device=dev)
        cols = newid[W.indices[pos].long()]
        keep = cols >= 0
        rows, cols, vals = rows[keep], cols[keep], W.values[pos][keep]
        indptr = torch.zeros(m + 1, dtype=torch.int64, device=dev)
        indptr[1:] = torch.cumsum(torch.bincount(rows, minlength=m), 0)
        return SparseSymmetricMatrix.from_device(DeviceCSR(indptr, cols.to(torch.int32), vals.contiguous(), (m, m)))

    def require_adjacency(self) -> None:
        if np.any(self.diagonal() != 0.0):
            raise ValueError("adjacency must have a zero diagonal")
        if self.nnz and float(self.csr.data.min()) < 0.0:
            raise ValueError("adjacency must be nonnegative")
