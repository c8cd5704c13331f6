"""Graph-side boundary of the hot path: degrees and symmetric normalisation.

``degrees`` / ``normalize_adjacency`` restate the reference
(``graph.py:118-139``) on the device (kernel K1): d = W 1 and
S_ij = (w_ij s_i) s_j with s = 1/sqrt(d), 0 where d == 0 -- the same
operation order as the reference, so S is bitwise equal in fp64.

``ComponentLabeling`` mirrors the reference container (``graph.py:168-212``)
because every ``SpectralDecomposition`` carries one; ``connected_components``
(``graph.py:215-250``) labels an adjacency on the device (kernel K11) for
``spectral.decompose_blockwise``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N
from .sparsemat import DeviceCSR, SparseSymmetricMatrix


@dataclass(frozen=True, eq=False)
class ComponentLabeling:
    labels: np.ndarray
    sizes: np.ndarray
    order: np.ndarray

    def __post_init__(self):
        labels = np.asarray(self.labels, dtype=np.int64)
        sizes = np.asarray(self.sizes, dtype=np.int64)
        order = np.asarray(self.order, dtype=np.int64)
        n = labels.shape[0]
        if order.shape != (n,) or not np.array_equal(np.sort(order), np.arange(n)):
            raise ValueError("order must be a permutation of 0..n-1")
        if int(sizes.sum()) != n:
            raise ValueError("component sizes must sum to n")
        object.__setattr__(self, "labels", labels)
        object.__setattr__(self, "sizes", sizes)
        object.__setattr__(self, "order", order)

    @classmethod
    def trivial(cls, n: int) -> "ComponentLabeling":
        return cls(np.zeros(n, dtype=np.int64), np.array([n], dtype=np.int64), np.arange(n))

    @property
    def n(self) -> int:
        return self.labels.shape[0]

    @property
    def count(self) -> int:
        return self.sizes.shape[0]

    def vertices_of(self, component: int) -> np.ndarray:
        return np.flatnonzero(self.labels == component)


def degrees_device(adjacency, device=None):
    """Row sums of the adjacency as a float64 CUDA tensor."""
    import torch

    A = SparseSymmetricMatrix.coerce(adjacency)
    W = A.device(torch.float64, device)
    ctx = N.Context.get(W.device)
    deg = torch.empty(A.n, dtype=torch.float64, device=W.device)
    ctx.call("csr_row_sums", A.n, N.ptr(W.indptr), N.ptr(W.values), N.ptr(deg))
    return deg


def degrees(adjacency) -> np.ndarray:
    """d = W 1 (``graph.py:118-121``), computed on the device."""
    A = SparseSymmetricMatrix.coerce(adjacency)
    if A._csr is not None:
        A.require_adjacency()
    return degrees_device(A).cpu().numpy()


def normalize_adjacency(adjacency, degree, dtype="float64", device=None) -> SparseSymmetricMatrix:
    """D^-1/2 W D^-1/2 with 0/0 = 0 (``graph.py:124-139``) on the device.

    Returns a device-resident ``SparseSymmetricMatrix`` (host copy on demand).
    """
    import torch

    A = SparseSymmetricMatrix.coerce(adjacency)
    if isinstance(degree, torch.Tensor):
        deg = degree.to(dtype=torch.float64)
    else:
        degree = np.asarray(degree, dtype=np.float64)
        if degree.shape != (A.n,):
            raise ValueError("degree vector shape does not match adjacency")
        deg = torch.as_tensor(degree)
    W = A.device(torch.float64, device)
    deg = deg.to(W.device)
    ctx = N.Context.get(W.device)
    dt = N.torch_dtype(dtype)
    out = torch.empty(W.nnz, dtype=dt, device=W.device)
    ctx.call("csr_normalize", N.dtype_code(dt), A.n, 0, N.ptr(W.indptr), N.ptr(W.indices), N.ptr(W.values),
             N.ptr(deg), N.ptr(out))
    return SparseSymmetricMatrix.from_device(DeviceCSR(W.indptr, W.indices, out, W.shape))


def connected_components(adjacency) -> ComponentLabeling:
    """Connected components ordered by decreasing size, ties by the smallest
    vertex index (``graph.py:215-250``); isolated vertices are singletons.

    The roots (smallest vertex of each component) come from the K11 kernel;
    numbering, sizes and the block order follow the reference's rules.
    """
    import torch

    A = SparseSymmetricMatrix.coerce(adjacency)
    if A._csr is not None:
        A.require_adjacency()
    W = A.device(torch.float64)
    n = A.n
    roots = torch.empty(n, dtype=torch.int64, device=W.device)
    N.Context.get(W.device).call("connected_components", n, N.ptr(W.indptr), N.ptr(W.indices), N.ptr(roots),
                                 N.ptr(None))
    uniq, inverse, counts = torch.unique(roots, sorted=True, return_inverse=True, return_counts=True)
    rank = torch.argsort(-counts, stable=True)          # size desc, then smallest root (uniq is ascending)
    label_of = torch.empty_like(rank)
    label_of[rank] = torch.arange(rank.numel(), device=rank.device)
    labels = label_of[inverse]
    order = torch.argsort(labels, stable=True)          # ascending vertex index inside each block
    return ComponentLabeling(labels.cpu().numpy(), counts[rank].cpu().numpy(), order.cpu().numpy())
