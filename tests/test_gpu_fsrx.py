"""FSRX round trip of device decompositions: a float32
decomposition written and read back answers queries with bit-identical scores
and top-k; the component labeling and metadata survive."""

import numpy as np
import pytest
import scipy.sparse as sp

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1703_06935_b200 import fsrx, graph, ranking, spectral  # noqa: E402
from paper_1703_06935_b200.sparsemat import SparseSymmetricMatrix  # noqa: E402


@pytest.fixture(scope="module")
def c1(golden):
    g = golden("c1")
    n, r, p, q, tau, seed = (int(v) for v in g["params"])
    S = SparseSymmetricMatrix(sp.csr_matrix((g["S_data"], g["W_indices"], g["W_indptr"]), shape=(n, n)))
    dec = spectral.decompose(S, r, p=p, q=q, seed=seed, dtype="float32")
    batch = ranking.QueryBatch(n, g["y_ptr"], g["y_idx"], g["y_val"])
    return dec, spectral.sparsify(dec, tau), batch


@pytest.mark.parametrize("which", ["dense", "sparse"])
def test_round_trip_scores_bit_identical(tmp_path, c1, which):
    dec, sdec, batch = c1
    d = dec if which == "dense" else sdec
    path = tmp_path / "dec.fsrx"
    fsrx.save_decomposition(d, path, alpha_hint=0.99)
    back = fsrx.load_decomposition(path)
    assert back.variant is d.variant and back.is_sparse == d.is_sparse
    np.testing.assert_array_equal(back.eigenvalues, d.eigenvalues)
    assert back.provenance.seed == d.provenance.seed
    h = ranking.h_alpha(0.99)
    X0 = ranking.filter_batch(d, h, batch)
    X1 = ranking.filter_batch(back, h, batch)
    np.testing.assert_array_equal(X0, X1)
    i0, v0 = ranking.top_k(d, h, batch, k=100)
    i1, v1 = ranking.top_k(back, h, batch, k=100)
    np.testing.assert_array_equal(i0, i1)
    np.testing.assert_array_equal(v0, v1)


def test_blockwise_labeling_survives(tmp_path, golden):
    b = golden("blockwise")
    n = b["labels"].size
    W = SparseSymmetricMatrix(sp.csr_matrix((b["W_data"], b["W_indices"], b["W_indptr"]), shape=(n, n)))
    S = SparseSymmetricMatrix(sp.csr_matrix((b["S_data"], b["W_indices"], b["W_indptr"]), shape=(n, n)))
    lab = graph.connected_components(W)
    dec = spectral.decompose_blockwise(S, lab, r=20, rho=50, p=10, q=4, seed=7, dtype="float32")
    path = tmp_path / "bw.fsrx"
    fsrx.save_decomposition(dec, path)
    back = fsrx.load_decomposition(path)
    np.testing.assert_array_equal(back.components.labels, lab.labels)
    np.testing.assert_array_equal(back.components.sizes, lab.sizes)
    np.testing.assert_array_equal(back.components.order, lab.order)
    np.testing.assert_array_equal(back.U_device.cpu().numpy(), dec.U_device.cpu().numpy())
