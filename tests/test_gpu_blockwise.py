"""Device connected components (K11) and the blockwise / exact decompositions
(reference graph.py:215-250, spectral.py:200-266,
312-390) against the reference's own outputs (tests/golden/blockwise.npz).

Labels, sizes and block order are integer results: identical.  Spectral
results are compared through invariants that do not depend on the order of
(numerically) equal eigenvalues or on eigenvector signs -- U diag(lam) U^T,
U U^T and eta -- in fp64 to 1e-9, plus the variant.  For components with
distinct eigenvalues the sign-fixed vectors are compared directly.
"""

import numpy as np
import pytest
import scipy.sparse as sp

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import fsr_oracle as O  # noqa: E402
from paper_1703_06935_b200 import graph, spectral  # noqa: E402
from paper_1703_06935_b200.sparsemat import SparseSymmetricMatrix  # noqa: E402


@pytest.fixture(scope="module")
def bw(golden):
    b = golden("blockwise")
    n = b["labels"].size
    W = sp.csr_matrix((b["W_data"], b["W_indices"], b["W_indptr"]), shape=(n, n))
    S = sp.csr_matrix((b["S_data"], b["W_indices"], b["W_indptr"]), shape=(n, n))
    return b, SparseSymmetricMatrix(W), SparseSymmetricMatrix(S)


def same_operator(U, lam, U_ref, lam_ref, tol):
    np.testing.assert_allclose(np.sort(lam)[::-1], np.sort(lam_ref)[::-1], atol=tol)
    np.testing.assert_allclose((U * lam) @ U.T, (U_ref * lam_ref) @ U_ref.T, atol=tol)
    np.testing.assert_allclose(U @ U.T, U_ref @ U_ref.T, atol=tol)


def test_components_match_reference(bw):
    b, W, _ = bw
    lab = graph.connected_components(W)
    np.testing.assert_array_equal(lab.labels, b["labels"])
    np.testing.assert_array_equal(lab.sizes, b["sizes"])
    np.testing.assert_array_equal(lab.order, b["order"])


@pytest.mark.parametrize("case", ["path", "star", "empty", "random"])
def test_components_vs_oracle(case):
    rng = np.random.default_rng(3)
    if case == "path":  # long chain in shuffled order: many hook/jump rounds
        n = 5000
        p = rng.permutation(n)
        r, c = p[:-1], p[1:]
    elif case == "star":
        n = 3000
        r, c = np.zeros(n - 1, dtype=np.int64) + n - 1, np.arange(n - 1)
    elif case == "empty":
        n = 50
        r = c = np.zeros(0, dtype=np.int64)
    else:
        n = 20000
        m = 12000  # below the percolation threshold: many components of all sizes
        r, c = rng.integers(0, n, m), rng.integers(0, n, m)
        keep = r != c
        r, c = r[keep], c[keep]
    W = sp.coo_matrix((np.ones(2 * r.size), (np.r_[r, c], np.r_[c, r])), shape=(n, n)).tocsr()
    W.data[:] = 1.0
    lab = graph.connected_components(SparseSymmetricMatrix(W))
    labels, sizes, order = O.connected_components(W)
    np.testing.assert_array_equal(lab.labels, labels)
    np.testing.assert_array_equal(lab.sizes, sizes)
    np.testing.assert_array_equal(lab.order, order)


def test_submatrix_matches_scipy(bw):
    _, _, S = bw
    idx = np.sort(np.random.default_rng(0).choice(S.n, 173, replace=False))
    sub = S.submatrix(idx).csr
    ref = sp.csr_matrix(S.csr[idx][:, idx])
    ref.sort_indices()
    assert (sub != ref).nnz == 0
    np.testing.assert_array_equal(sub.indptr, ref.indptr)


@pytest.mark.parametrize("tag,rho", [("mixed", 50), ("exact", 400)])
def test_blockwise_matches_reference(bw, tag, rho):
    b, W, S = bw
    lab = graph.connected_components(W)
    dec = spectral.decompose_blockwise(S, lab, r=int(b[f"{tag}_r"]), rho=rho, p=10, q=4, seed=7)
    assert dec.variant.value == str(b[f"{tag}_variant"])
    same_operator(dec.dense_u(), dec.eigenvalues, b[f"{tag}_U"], b[f"{tag}_lam"], 1e-9)
    np.testing.assert_allclose(dec.eta, b[f"{tag}_eta"], atol=1e-9)
    assert dec.components is lab


def test_exact_and_rank_r_match_reference(bw):
    b, W, S = bw
    lab = graph.connected_components(W)
    sub = W.submatrix(lab.vertices_of(2))
    Ssub = graph.normalize_adjacency(sub, graph.degrees(sub))
    ex = spectral.exact_eigendecomposition(Ssub)
    assert ex.variant is spectral.Variant.EXACT
    np.testing.assert_allclose(ex.eigenvalues, b["exact_sub_lam"], atol=1e-12)
    # distinct eigenvalues: sign-fixed eigenvectors agree column by column
    gaps = np.diff(b["exact_sub_lam"])
    assert np.all(np.abs(gaps) > 1e-8)
    np.testing.assert_allclose(ex.U, b["exact_sub_U"], atol=1e-10)
    rr = spectral.rank_r_decomposition(S.submatrix(lab.vertices_of(1)), 17)
    assert rr.variant is spectral.Variant.RANK_R
    np.testing.assert_allclose(rr.eigenvalues, b["rankr_lam"], atol=1e-12)
    np.testing.assert_allclose(rr.U, b["rankr_U"], atol=1e-10)
    np.testing.assert_allclose(rr.eta, b["rankr_eta"], atol=1e-10)
    tr = spectral.truncate_rank(rr, 5)
    assert tr.variant is spectral.Variant.RANK_R and tr.r == 5
    np.testing.assert_allclose(tr.U, b["rankr_U"][:, :5], atol=1e-10)


def test_blockwise_float32_invariants(bw):
    b, W, S = bw
    lab = graph.connected_components(W)
    dec = spectral.decompose_blockwise(S, lab, r=int(b["mixed_r"]), rho=50, p=10, q=4, seed=7, dtype="float32")
    np.testing.assert_allclose(np.sort(dec.eigenvalues), np.sort(b["mixed_lam"]), atol=1e-5)
    np.testing.assert_allclose(dec.eta, b["mixed_eta"], atol=1e-4)


def test_blockwise_errors(bw):
    b, W, S = bw
    lab = graph.connected_components(W)
    with pytest.raises(ValueError):
        spectral.decompose_blockwise(S, lab, r=0, rho=5)
    with pytest.raises(ValueError):
        spectral.decompose_blockwise(S, lab, r=5, rho=0)
    with pytest.raises(ValueError):
        spectral.decompose_blockwise(S, graph.ComponentLabeling.trivial(3), r=5, rho=5)
    with pytest.raises(spectral.NumericalError):
        spectral.exact_eigendecomposition(S, max_n=10)
    with pytest.raises(ValueError):
        spectral.truncate_rank(spectral.exact_eigendecomposition(S.submatrix(lab.vertices_of(3))), 0)
