"""tcgen05 3xTF32 dense kernels (Gram, cross, R^-1 apply, lift) vs fp64 numpy.

Tolerances: the 3xTF32 split recovers ~fp32 accuracy; results are compared
normwise (max |err| / max |ref|) at <= 2e-6, the 1xTF32 Gram at <= 2e-3.
"""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1703_06935_b200 import _native as N  # noqa: E402
from paper_1703_06935_b200 import spectral  # noqa: E402

SHAPES = [(1000, 8), (3000, 100), (5000, 350), (4099, 257), (20000, 520), (2049, 1)]


def rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


@pytest.fixture(params=["auto", "cublas"])
def ctx(request):
    c = N.Context.get()
    c.set_dense_path(request.param)
    yield c
    c.set_dense_path("auto")


@pytest.mark.parametrize("n,k", SHAPES)
def test_gram(ctx, n, k):
    rng = np.random.default_rng(n + k)
    A = rng.standard_normal((n, k)).astype(np.float32)
    Ad = torch.as_tensor(A).cuda()
    G = torch.empty(k, k, dtype=torch.float64, device="cuda")
    ctx.call("gram", N.F32, n, k, N.ptr(Ad), k, N.ptr(G), 0)
    ref = A.astype(np.float64).T @ A.astype(np.float64)
    assert rel(G.cpu().numpy(), ref) < 2e-6
    np.testing.assert_array_equal(G.cpu().numpy(), G.cpu().numpy().T)
    # accumulate doubles it
    ctx.call("gram", N.F32, n, k, N.ptr(Ad), k, N.ptr(G), 1)
    assert rel(G.cpu().numpy(), 2 * ref) < 2e-6


@pytest.mark.parametrize("n,k", SHAPES[:4])
def test_gram_fast(n, k):
    ctx = N.Context.get()
    rng = np.random.default_rng(7)
    A = rng.standard_normal((n, k)).astype(np.float32)
    Ad = torch.as_tensor(A).cuda()
    G = torch.empty(k, k, dtype=torch.float64, device="cuda")
    ctx.call("gram_tf32", n, k, N.ptr(Ad), k, N.ptr(G), 0, 1)
    ref = A.astype(np.float64).T @ A.astype(np.float64)
    assert rel(G.cpu().numpy(), ref) < 2e-3


@pytest.mark.parametrize("n,k", SHAPES)
def test_cross(ctx, n, k):
    rng = np.random.default_rng(3 * n + k)
    Q = rng.standard_normal((n, k)).astype(np.float32)
    B = rng.standard_normal((n, k)).astype(np.float32)
    C = torch.empty(k, k, dtype=torch.float64, device="cuda")
    Qd, Bd = torch.as_tensor(Q).cuda(), torch.as_tensor(B).cuda()
    ctx.call("cross", N.F32, n, k, N.ptr(Qd), k, N.ptr(Bd), k, N.ptr(C), 0)
    ref = Q.astype(np.float64).T @ B.astype(np.float64)
    got = C.cpu().numpy()
    # layout: either Q^T B or its transpose (callers symmetrise)
    assert min(rel(got, ref), rel(got.T, ref)) < 2e-6


@pytest.mark.parametrize("n,k", SHAPES)
def test_apply_rinv(ctx, n, k):
    rng = np.random.default_rng(n * 7 + k)
    B = rng.standard_normal((n, k)).astype(np.float32)
    G = B.astype(np.float64).T @ B.astype(np.float64)
    R = np.linalg.cholesky(G).T  # upper
    Rd = torch.as_tensor(np.asfortranarray(R).ravel(order="F").copy()).cuda()  # column-major R
    Bd = torch.as_tensor(B).cuda()
    ctx.call("apply_rinv", N.F32, n, k, N.ptr(Rd), N.ptr(Bd), k)
    ref = np.linalg.solve(R.T, B.astype(np.float64).T).T
    assert rel(Bd.cpu().numpy(), ref) < 5e-6


@pytest.mark.parametrize("n,k,r", [(3000, 100, 60), (5000, 350, 300), (4099, 257, 250), (2000, 40, 40)])
def test_lift(ctx, n, k, r):
    rng = np.random.default_rng(n + 3 * k + r)
    Q = rng.standard_normal((n, k)).astype(np.float32)
    V = rng.standard_normal((k, r))
    U = torch.empty(n, r, dtype=torch.float32, device="cuda")
    Qd, Vd = torch.as_tensor(Q).cuda(), torch.as_tensor(V).cuda()
    ctx.call("lift", N.F32, n, k, r, N.ptr(Qd), k, N.ptr(Vd), N.ptr(U), r)
    ref = Q.astype(np.float64) @ V
    assert rel(U.cpu().numpy(), ref) < 2e-6


def test_orthonormalize_fp32_tc():
    rng = np.random.default_rng(1)
    Y0 = rng.standard_normal((30000, 600))
    Y = torch.as_tensor(Y0).to("cuda", torch.float32)
    spectral.orthonormalize(Y)
    Q = Y.double().cpu().numpy()
    assert np.abs(Q.T @ Q - np.eye(600)).max() < 5e-6
