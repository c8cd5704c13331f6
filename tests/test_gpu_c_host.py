"""The C boundary from a C host: tests/c_host/fsr_host_demo.c is compiled
with gcc against include/fsr.h and libfsr.so, runs decompose -> sparsify ->
filter + rank through the operator-level calls (fsr_decompose,
fsr_sparsify_select / fsr_sparsify_apply, fsr_filter_batch), and its outputs
are checked against the oracle: Ritz values <= 1e-10 normwise (fp64 parity
mode), the kept count, eta of the sparse U~, and the top-k of one query."""

import os
import shutil
import subprocess

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import fsr_oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def build_demo(tmp_path):
    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("gcc not available")
    from paper_1703_06935_b200 import _native

    libdir = os.path.dirname(_native.LIB_PATH)
    cuda = "/usr/local/cuda"
    exe = str(tmp_path / "fsr_host_demo")
    cmd = [gcc, "-O2", "-std=c11", os.path.join(REPO, "tests", "c_host", "fsr_host_demo.c"), "-o", exe,
           "-I", os.path.join(REPO, "include"), "-I", os.path.join(cuda, "include"), "-L", libdir, "-lfsr",
           "-L", os.path.join(cuda, "lib64"), "-lcudart", f"-Wl,-rpath,{libdir}", f"-Wl,-rpath,{cuda}/lib64"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_c_host_decompose_sparsify_filter(tmp_path):
    rng = np.random.default_rng(11)
    n, r, p, q, tau, topk = 600, 16, 8, 3, 2400, 25
    M = rng.random((n, n)) * (rng.random((n, n)) < 0.02)
    M = np.triu(M, 1)
    W = sp.csr_matrix(M + M.T)
    S = O.normalize_adjacency(W, O.degrees(W))
    S.sort_indices()
    y_idx = np.array([4, 77, 310, 599], dtype=np.int64)
    y_val = np.array([1.0, 0.5, 0.25, 0.125])
    U_ref, lam_ref, _ = O.decompose(S, r, p=p, q=q, seed=0)
    w = O.transfer_values(O.h_alpha(0.99), lam_ref)
    src = tmp_path / "in.bin"
    with open(src, "wb") as f:
        np.array([n, S.nnz, y_idx.size], dtype=np.int64).tofile(f)
        S.indptr.astype(np.int64).tofile(f)
        S.indices.astype(np.int32).tofile(f)
        S.data.astype(np.float64).tofile(f)
        y_idx.tofile(f)
        y_val.tofile(f)
        w.astype(np.float64).tofile(f)
    exe = build_demo(tmp_path)
    out = tmp_path / "out.bin"
    res = subprocess.run([exe, str(src), str(out), str(r), str(p), str(q), str(tau), str(topk)],
                         capture_output=True, text=True, timeout=300)
    assert res.returncode == 0, res.stderr
    raw = np.fromfile(out, dtype=np.float64)
    lam = raw[:r]
    eta = raw[r:r + n]
    kept = int(np.frombuffer(raw[r + n:r + n + 1].tobytes(), dtype=np.int64)[0])
    ti = np.frombuffer(raw[r + n + 1:r + n + 1 + topk].tobytes(), dtype=np.int64)
    tv = raw[r + n + 1 + topk:]
    assert np.abs(lam - lam_ref).max() <= 1e-10 * np.abs(lam_ref).max()
    Ut, eta_s = O.sparsify(U_ref, tau)
    assert kept == Ut.nnz
    np.testing.assert_allclose(eta, eta_s, rtol=1e-9, atol=1e-12)
    x = O.filter_scores(Ut, lam_ref, eta_s, w, y_idx, y_val)
    order = O.rank(x)[:topk]
    np.testing.assert_array_equal(ti, order)
    np.testing.assert_allclose(tv, x[order], rtol=1e-9, atol=1e-12)
    assert "cholqr2" in res.stdout  # the fp64 schedule: CholeskyQR2 every round
