"""B200-native fast spectral ranking (FSR, arXiv 1703.06935) hot path.

Reference-compatible entry points (reference: /root/reference/pkg/src/specrank):

* ``spectral``: gaussian_matrix, range_finder, approx_eigendecomposition,
  decompose, sparsify, RangeBasis, SpectralDecomposition, Variant, Provenance,
  NumericalError
* ``ranking``: TransferFunction, h_alpha, custom_transfer, ObservationVector,
  filter, filter_batch, rank
* ``graph``: degrees, normalize_adjacency, ComponentLabeling
* ``sparsemat``: SparseSymmetricMatrix

All arithmetic runs in libfsr.so (include/fsr.h), hand-written CUDA for sm_100a.
"""

__version__ = "0.1.0"
