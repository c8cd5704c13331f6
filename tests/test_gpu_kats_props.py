"""The SPEC known-answer tests for `filter` and the property tests of the
build's test plan, on the device.

KATs (on an EXACT decomposition of a random normalised
adjacency, fp64):
  * h_alpha(0) (h == 1) gives x = y;
  * h_alpha(0.99) matches the dense (1 - alpha)(I - alpha W)^-1 y to 1e-6;
  * the identity transfer gives x = W y;
  * filter is linear to 1e-10.
Properties (hypothesis, random small symmetric CSR): linearity, invariance to
column signs of U, tau >= nnz(U) leaves U unchanged; an empty observation
gives zero scores.  Online-only parity (item 3): the oracle's filter on the
device-produced U~ equals the device filter (support-aligned).
"""

import numpy as np
import pytest
import scipy.sparse as sp

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from hypothesis import HealthCheck, given, settings  # noqa: E402
from hypothesis import strategies as st  # noqa: E402

from oracle import fsr_oracle as O  # noqa: E402
from paper_1703_06935_b200 import graph, ranking, spectral  # noqa: E402
from paper_1703_06935_b200.sparsemat import SparseSymmetricMatrix  # noqa: E402


def random_adjacency(n, density, seed):
    rng = np.random.default_rng(seed)
    M = sp.random(n, n, density=density, random_state=rng, format="csr")
    W = M + M.T
    W.setdiag(0.0)
    W.eliminate_zeros()
    W.sort_indices()
    return W


def normalized(W):
    A = SparseSymmetricMatrix.from_scipy(W)
    return graph.normalize_adjacency(A, graph.degrees(A))


def ovec(n, idx, val):
    idx = np.asarray(idx, dtype=np.int64)
    o = np.argsort(idx)
    return ranking.ObservationVector(n, idx[o], np.asarray(val, dtype=np.float64)[o], cap=max(1, len(idx)))


@pytest.fixture(scope="module")
def exact64():
    W = random_adjacency(120, 0.08, 3)
    S = normalized(W)
    return S, spectral.exact_eigendecomposition(S)


def test_kat_h0_gives_identity(exact64):
    S, dec = exact64
    n = S.n
    y = ovec(n, [3, 17, 64, 99], [0.5, 1.0, 0.25, 2.0])
    x = ranking.filter(dec, ranking.h_alpha(0.0), y, copy_uncovered=False)
    np.testing.assert_allclose(x, y.to_dense(), atol=1e-10)


def test_kat_h_alpha_matches_dense_solve(exact64):
    S, dec = exact64
    n = S.n
    alpha = 0.99
    y = ovec(n, [1, 2, 50, 77], [1.0, 0.3, 0.7, 0.2])
    x = ranking.filter(dec, ranking.h_alpha(alpha), y, copy_uncovered=False)
    ref = (1.0 - alpha) * np.linalg.solve(np.eye(n) - alpha * S.to_dense(), y.to_dense())
    np.testing.assert_allclose(x, ref, atol=1e-6 * np.abs(ref).max())


def test_kat_identity_transfer_gives_wy(exact64):
    S, dec = exact64
    n = S.n
    ident = ranking.custom_transfer(lambda v: v, nondecreasing=True, name="identity")
    y = ovec(n, [0, 10, 20], [1.0, 2.0, 3.0])
    x = ranking.filter(dec, ident, y, copy_uncovered=False)
    np.testing.assert_allclose(x, S.csr @ y.to_dense(), atol=1e-10)


def test_kat_linearity(exact64):
    S, dec = exact64
    n = S.n
    h = ranking.h_alpha(0.9)
    y1 = ovec(n, [4, 9, 33], [1.0, 0.5, 0.25])
    y2 = ovec(n, [9, 40], [2.0, 1.5])
    yc = ranking.ObservationVector.from_dense(0.7 * y1.to_dense() + 1.3 * y2.to_dense())
    x1, x2, xc = (ranking.filter(dec, h, y, copy_uncovered=False) for y in (y1, y2, yc))
    np.testing.assert_allclose(xc, 0.7 * x1 + 1.3 * x2, atol=1e-10 * np.abs(xc).max())


def test_empty_observation_gives_zero_scores(exact64):
    S, dec = exact64
    y = ranking.ObservationVector(S.n, np.zeros(0, np.int64), np.zeros(0), cap=5)
    x = ranking.filter(dec, ranking.h_alpha(0.99), y)
    assert x.shape == (S.n,) and not np.any(x)


def test_online_only_parity_on_device_u(golden):
    """Support-aligned C5 parity: the oracle filter on the device-produced
    U~ (as host CSR float64) against the device filter, fp32 and fp64."""
    g = golden("c1")
    n, r, p, q, tau, seed = (int(v) for v in g["params"])
    S = SparseSymmetricMatrix(sp.csr_matrix((g["S_data"], g["W_indices"], g["W_indptr"]), shape=(n, n)))
    batch = ranking.QueryBatch(n, g["y_ptr"], g["y_idx"], g["y_val"])
    h = ranking.h_alpha(float(g["alpha"]))
    for dtype, tol in (("float64", 1e-12), ("float32", 1e-5)):
        dec = spectral.decompose(S, r, p=p, q=q, seed=seed, dtype=dtype)
        sdec = spectral.sparsify(dec, tau)
        X = ranking.filter_batch(sdec, h, batch)
        U = sdec.U.astype(np.float64)
        w = O.transfer_values(O.h_alpha(float(g["alpha"])), sdec.eigenvalues)
        for j in range(0, batch.b, 9):
            s, e = batch.y_ptr[j], batch.y_ptr[j + 1]
            ref = O.filter_scores(U, sdec.eigenvalues, sdec.eta, w, batch.y_idx[s:e], batch.y_val[s:e])
            assert np.linalg.norm(X[j] - ref) <= tol * np.linalg.norm(ref)


SETTINGS = settings(max_examples=8, deadline=None, suppress_health_check=[HealthCheck.too_slow])


@SETTINGS
@given(n=st.integers(20, 90), density=st.floats(0.05, 0.3), seed=st.integers(0, 10_000),
       q=st.integers(1, 4), data=st.data())
def test_property_filter_linear_and_sign_invariant(n, density, seed, q, data):
    W = random_adjacency(n, density, seed)
    if W.nnz == 0:
        return
    S = normalized(W)
    r_hat = data.draw(st.integers(2, n))
    r = data.draw(st.integers(1, r_hat))
    dec = spectral.decompose(S, r, p=r_hat - r, q=q, seed=seed)
    h = ranking.h_alpha(0.9)
    rng = np.random.default_rng(seed)
    i1 = rng.choice(n, size=min(5, n), replace=False)
    i2 = rng.choice(n, size=min(4, n), replace=False)
    y1, y2 = ovec(n, i1, rng.random(i1.size)), ovec(n, i2, rng.random(i2.size))
    yc = ranking.ObservationVector.from_dense(2.0 * y1.to_dense() + 0.5 * y2.to_dense())
    x1, x2, xc = (ranking.filter(dec, h, y, copy_uncovered=False) for y in (y1, y2, yc))
    scale = max(np.abs(xc).max(), 1e-300)
    assert np.abs(xc - (2.0 * x1 + 0.5 * x2)).max() <= 1e-10 * scale
    # flipping column signs of U leaves U h(Lambda) U^T unchanged
    flip = np.where(rng.random(dec.r) < 0.5, -1.0, 1.0)

    class Flipped:
        U = dec.U * flip
        eigenvalues = dec.eigenvalues
        eta = dec.eta
        variant = dec.variant
        provenance = dec.provenance
        components = dec.components

    xf = ranking.filter(Flipped, h, y1, copy_uncovered=False)
    assert np.abs(xf - x1).max() <= 1e-12 * max(np.abs(x1).max(), 1e-300)


@SETTINGS
@given(n=st.integers(10, 60), r=st.integers(1, 10), seed=st.integers(0, 10_000))
def test_property_tau_at_least_nnz_keeps_u(n, r, seed):
    W = random_adjacency(n, 0.2, seed)
    if W.nnz == 0:
        return
    S = normalized(W)
    r = min(r, n)
    dec = spectral.decompose(S, r, p=min(5, n - r), q=2, seed=seed)
    U = dec.U
    sdec = spectral.sparsify(dec, n * r + 3)
    np.testing.assert_array_equal(sdec.U.toarray(), U)
    np.testing.assert_allclose(sdec.eta, dec.eta, rtol=1e-14)
