"""tcgen05 int8-Ozaki dense kernels (Gram, cross, R^-1 apply, lift) vs fp64 numpy.

Tolerances (normwise: max |err| / max |ref|): the cuBLAS path (fp64 upcast /
fp32 TRSM, SGEMM) <= 2e-6.  The tensor-core path slices every value into 21
fixed-point bits below a shared exponent (per reduction vector) and
accumulates exactly in int32: its error is unbiased, ~2^-21 of the vector
maxima per product.  Incoherent random sums (these tests) see up to ~4e-5;
the coherent sums of the actual pipeline (Gram of a near-orthonormal block,
C = Q^T A Q ~ diag(lambda)) see ~1e-7.
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


TOL = {"auto": 5e-5, "cublas": 2e-6}


@pytest.fixture(params=["auto", "cublas"])
def ctx(request):
    c = N.Context.get()
    c.set_dense_path(request.param)
    c.path = request.param
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
    assert rel(G.cpu().numpy(), ref) < 2e-6  # coherent diagonal dominates
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
    ctx.call("gram_levels", n, k, N.ptr(Ad), k, N.ptr(G), 0, 1)
    ref = A.astype(np.float64).T @ A.astype(np.float64)
    assert rel(G.cpu().numpy(), ref) < 5e-2  # one 7-bit slice: a preconditioner, not a Gram


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
    assert min(rel(got, ref), rel(got.T, ref)) < TOL[ctx.path]


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
    assert rel(Bd.cpu().numpy(), ref) < 2 * TOL[ctx.path] + 3e-6


@pytest.mark.parametrize("n,k,r", [(3000, 100, 60), (5000, 350, 300), (4099, 257, 250), (2000, 40, 40)])
def test_lift(ctx, n, k, r):
    rng = np.random.default_rng(n + 3 * k + r)
    Q = rng.standard_normal((n, k)).astype(np.float32)
    V = rng.standard_normal((k, r))
    U = torch.empty(n, r, dtype=torch.float32, device="cuda")
    Qd, Vd = torch.as_tensor(Q).cuda(), torch.as_tensor(V).cuda()
    ctx.call("lift", N.F32, n, k, r, N.ptr(Qd), k, N.ptr(Vd), N.ptr(U), r)
    ref = Q.astype(np.float64) @ V
    assert rel(U.cpu().numpy(), ref) < TOL[ctx.path]


def test_orthonormalize_fp32_tc():
    rng = np.random.default_rng(1)
    Y0 = rng.standard_normal((30000, 600))
    Y = torch.as_tensor(Y0).to("cuda", torch.float32)
    spectral.orthonormalize(Y)
    Q = Y.double().cpu().numpy()
    assert np.abs(Q.T @ Q - np.eye(600)).max() < 5e-6


def test_pipeline_cross_is_accurate():
    # the Rayleigh-Ritz cross product on an orthonormal Q and B = A Q (coherent sums)
    rng = np.random.default_rng(4)
    Q = np.linalg.qr(rng.standard_normal((50000, 300)))[0]
    lam = np.linspace(1.0, 0.1, 300)
    B = Q * lam + 1e-3 * rng.standard_normal(Q.shape) / np.sqrt(Q.shape[0])
    Qd = torch.as_tensor(Q).to("cuda", torch.float32)
    Bd = torch.as_tensor(B).to("cuda", torch.float32)
    C = torch.empty(300, 300, dtype=torch.float64, device="cuda")
    N.Context.get().call("cross", N.F32, 50000, 300, N.ptr(Qd), 300, N.ptr(Bd), 300, N.ptr(C), 0)
    ref = Qd.double().cpu().numpy().T @ Bd.double().cpu().numpy()
    got = C.cpu().numpy()
    assert min(rel(got, ref), rel(got.T, ref)) < 1e-6
