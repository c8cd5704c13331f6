"""Per-kernel parity of the CUDA path against the oracle and the golden fixtures.

Tolerances: integer/index work is bit-exact; fp64 kernels are bitwise where
the reference order is reproduced (K1 normalisation, K2 SpMM) and within
stated relative bounds elsewhere; fp32 kernels within 1e-5 relative.
"""

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import fsr_oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1703_06935_b200 import _native as N  # noqa: E402
from paper_1703_06935_b200 import graph, ranking, spectral  # noqa: E402
from paper_1703_06935_b200.sparsemat import SparseSymmetricMatrix  # noqa: E402


def c1_mats(g):
    n = int(g["params"][0])
    W = sp.csr_matrix((g["W_data"], g["W_indices"], g["W_indptr"]), shape=(n, n))
    S = sp.csr_matrix((g["S_data"], g["W_indices"], g["W_indptr"]), shape=(n, n))
    return W, S


# ---------------------------------------------------------------- K0 -------
def test_gaussian_matches_reference(golden):
    g = golden("gaussian")
    for i in range(int(g["count"])):
        r, c, s = (int(v) for v in g[f"g{i}_shape"])
        ref = g[f"g{i}"]
        out = spectral.gaussian_matrix(r, c, s).cpu().numpy()
        np.testing.assert_allclose(out, ref, rtol=4e-15, atol=4e-15)
        out32 = spectral.gaussian_matrix(r, c, s, dtype="float32").cpu().numpy()
        np.testing.assert_array_equal(out32, ref.astype(np.float32))


@pytest.mark.parametrize("rows,cols", [(37, 11), (64, 10), (5, 3), (1000, 7)])
def test_gaussian_row_shards_compose(rows, cols):
    full = spectral.gaussian_matrix(rows, cols, 99).cpu().numpy()
    ref = O.gaussian_matrix(rows, cols, 99)
    np.testing.assert_allclose(full, ref, rtol=4e-15, atol=4e-15)
    cuts = sorted({0, rows, rows // 3, rows // 2, (2 * rows) // 3})
    parts = [spectral.gaussian_block(rows, cols, 99, a, b).cpu().numpy() for a, b in zip(cuts[:-1], cuts[1:])]
    np.testing.assert_array_equal(np.concatenate(parts), full)


# ---------------------------------------------------------------- K1 -------
def test_normalize_bitwise(golden):
    g = golden("c1")
    W, S = c1_mats(g)
    A = SparseSymmetricMatrix.from_scipy(W)
    deg = graph.degrees(A)
    np.testing.assert_array_equal(deg, O.degrees(W))
    Sd = graph.normalize_adjacency(A, deg)
    np.testing.assert_array_equal(Sd.csr.data, S.data)


# ---------------------------------------------------------------- K2 -------
@pytest.mark.parametrize("ncols", [1, 3, 8, 350, 517])
def test_spmm_fp64_bitwise(golden, ncols):
    g = golden("c1")
    _, S = c1_mats(g)
    A = SparseSymmetricMatrix.from_scipy(S)
    rng = np.random.default_rng(ncols)
    X = rng.standard_normal((S.shape[0], ncols))
    Ad = A.device(torch.float64)
    Xd = torch.as_tensor(X).cuda()
    Yd = torch.empty_like(Xd)
    ctx = N.Context.get()
    spectral._spmm(ctx, N.F64, Ad, Xd, Yd)
    ref = S @ X
    if ncols == 1:
        np.testing.assert_allclose(Yd.cpu().numpy(), ref, rtol=1e-14, atol=1e-15)
    else:
        np.testing.assert_array_equal(Yd.cpu().numpy(), ref)


@pytest.mark.parametrize("ncols", [1, 4, 350, 1030])
def test_spmm_fp32(golden, ncols):
    g = golden("c1")
    _, S = c1_mats(g)
    A = SparseSymmetricMatrix.from_scipy(S)
    rng = np.random.default_rng(ncols)
    X = rng.standard_normal((S.shape[0], ncols)).astype(np.float32)
    Xd = torch.as_tensor(X).cuda()
    Yd = torch.empty_like(Xd)
    spectral._spmm(N.Context.get(), N.F32, A.device(torch.float32), Xd, Yd)
    ref = S @ X.astype(np.float64)
    err = np.abs(Yd.cpu().numpy() - ref).max() / np.abs(ref).max()
    assert err < 1e-6


@pytest.mark.parametrize("panel", [0, 32, 64, 128])
def test_spmm_empty_rows(panel):
    # rows with no nonzeros (isolated vertices) must produce exact zeros
    S = sp.csr_matrix((np.array([0.5, 0.5]), (np.array([0, 3]), np.array([3, 0]))), shape=(5, 5))
    A = SparseSymmetricMatrix.from_scipy(S)
    X = torch.arange(5 * 8, dtype=torch.float64, device="cuda").reshape(5, 8)
    Y = torch.full_like(X, 7.0)
    ctx = N.Context.get()
    ctx.set_spmm_panel(panel)
    try:
        spectral._spmm(ctx, N.F64, A.device(torch.float64), X, Y)
    finally:
        ctx.set_spmm_panel(0)
    np.testing.assert_array_equal(Y.cpu().numpy(), S @ X.cpu().numpy())


@pytest.mark.parametrize("panel", [32, 64, 128])
@pytest.mark.parametrize("ncols", [8, 350, 520])
def test_spmm_l2panel_schedule(golden, panel, ncols):
    """The L2-panel schedule keeps CSR order per element: fp64 bitwise equal to
    scipy, fp32 bitwise equal to the wide row-panel kernel."""
    g = golden("c1")
    _, S = c1_mats(g)
    A = SparseSymmetricMatrix.from_scipy(S)
    rng = np.random.default_rng(ncols + panel)
    X = rng.standard_normal((S.shape[0], ncols))
    ctx = N.Context.get()
    out = {}
    for dt, tdt in ((N.F64, torch.float64), (N.F32, torch.float32)):
        Xd = torch.as_tensor(X).to(tdt).cuda()
        for p in (0, panel):
            Yd = torch.full_like(Xd, float("nan"))
            ctx.set_spmm_panel(p)
            try:
                spectral._spmm(ctx, dt, A.device(tdt), Xd, Yd)
            finally:
                ctx.set_spmm_panel(0)
            out[(dt, p)] = Yd.cpu().numpy()
    np.testing.assert_array_equal(out[(N.F64, panel)], S @ X)
    np.testing.assert_array_equal(out[(N.F32, panel)], out[(N.F32, 0)])


def test_spmm_panel_option_rejects_bad_width():
    with pytest.raises(ValueError):
        N.Context.get().set_spmm_panel(48)


# ------------------------------------------------------------- K3-K6 -------
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_orthonormalize(dtype):
    rng = np.random.default_rng(1)
    Y0 = rng.standard_normal((3000, 120))
    Y = torch.as_tensor(Y0).to("cuda", N.torch_dtype(dtype))
    spectral.orthonormalize(Y)
    Q = Y.double().cpu().numpy()
    tol = 1e-13 if dtype == "float64" else 5e-6  # fp32 mode: 21-bit Ozaki slices
    assert np.abs(Q.T @ Q - np.eye(120)).max() < tol
    Qh = np.linalg.qr(Y0)[0]
    # same span, columns equal up to sign (CholeskyQR vs Householder)
    s = np.sign(np.sum(Q * Qh, axis=0))
    assert np.abs(Q - Qh * s).max() < (1e-10 if dtype == "float64" else 1e-4)


def test_orthonormalize_rank_deficient_falls_back():
    rng = np.random.default_rng(2)
    X = rng.standard_normal((200, 3))
    Y0 = X @ rng.standard_normal((3, 6))  # rank 3, six columns
    Y = torch.as_tensor(Y0).cuda()
    stats = []
    spectral.orthonormalize(Y, stats=stats)
    Q = Y.cpu().numpy()
    assert "householder" in stats[0]
    assert np.abs(Q.T @ Q - np.eye(6)).max() < 1e-8
    # range of the rank-3 input is contained in span(Q)
    P = Q @ Q.T
    assert np.abs(P @ X - X).max() < 1e-10


def test_kat_rank3_range_finder(golden):
    k = golden("kat")
    A = SparseSymmetricMatrix.from_dense(k["rank3_A"])
    basis = spectral.range_finder(A, 5, 3, 0)
    Q = basis.Q.cpu().numpy()
    resid = np.linalg.norm(k["rank3_A"] - Q @ (Q.T @ k["rank3_A"]), 2)
    assert resid < 1e-8


def test_kat_two_node(golden):
    k = golden("kat")
    A = SparseSymmetricMatrix.from_dense(np.array([[0.0, 1.0], [1.0, 0.0]]))
    dec = spectral.decompose(A, 2, p=0, q=3, seed=0)
    np.testing.assert_allclose(dec.eigenvalues, [1.0, -1.0], atol=1e-12)
    np.testing.assert_allclose(dec.U, k["two_U"], atol=1e-12)


@pytest.mark.parametrize("dtype,tol", [("float64", 1e-10), ("float32", 1e-5)])
def test_kat_random_decompose(golden, dtype, tol):
    k = golden("kat")
    A = SparseSymmetricMatrix.from_dense(k["rand_W_dense"])
    dec = spectral.decompose(A, 16, p=10, q=4, seed=3, dtype=dtype)
    lam = k["rand_lam"]
    assert np.abs(dec.eigenvalues - lam).max() <= tol * np.abs(lam).max()
    U = dec.U
    # column signs are fixed by the same rule; compare directly
    assert np.abs(U - k["rand_U"]).max() < (1e-8 if dtype == "float64" else 1e-4)
    np.testing.assert_allclose(dec.eta, k["rand_eta"], atol=tol * 10)


@pytest.mark.parametrize("dtype,tol", [("float64", 1e-10), ("float32", 1e-5)])
def test_kat_full_rank_reproduces_exact_spectrum(golden, dtype, tol):
    # q >= 8 with r_hat = n reproduces the exact eigenvalues
    k = golden("kat")
    A = SparseSymmetricMatrix.from_dense(k["rand_W_dense"])
    dec = spectral.decompose(A, 16, p=48, q=8, seed=3, dtype=dtype)
    ev = np.sort(np.linalg.eigvalsh(k["rand_W_dense"]))[::-1][:16]
    assert np.abs(dec.eigenvalues - ev).max() < tol
    U = dec.U
    # fp32 mode: 21-bit Ozaki slices in the dense stages
    assert np.abs(U.T @ U - np.eye(16)).max() < (1e-12 if dtype == "float64" else 1e-5)


def test_kat_random_sparsify_and_filter(golden):
    k = golden("kat")
    A = SparseSymmetricMatrix.from_dense(k["rand_W_dense"])
    dec = spectral.decompose(A, 16, p=10, q=4, seed=3)
    sdec = spectral.sparsify(dec, 200)
    coo = sdec.U.tocoo()
    flat = np.sort(coo.row.astype(np.int64) * 16 + coo.col)
    np.testing.assert_array_equal(flat, k["rand_sparse_flat"])
    np.testing.assert_allclose(sdec.eta, k["rand_sparse_eta"], rtol=1e-12)
    y = ranking.ObservationVector(64, k["rand_y_idx"], k["rand_y_val"], cap=4)
    h = ranking.h_alpha(0.99)
    np.testing.assert_allclose(ranking.filter(dec, h, y), k["rand_x_approx"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(ranking.filter(sdec, h, y), k["rand_x_sparse"], rtol=1e-9, atol=1e-12)
    heat = ranking.heat_kernel(10.0)
    np.testing.assert_allclose(ranking.filter(dec, heat, y), k["rand_x_heat"], rtol=1e-9, atol=1e-12)


def test_kat_isolated_vertex_copy_uncovered(golden):
    k = golden("kat")
    A = SparseSymmetricMatrix.from_dense(k["iso_W_dense"])
    dec = spectral.decompose(A, 6, p=2, q=3, seed=1)
    np.testing.assert_allclose(dec.eigenvalues, k["iso_lam"], atol=1e-12)
    sdec = spectral.sparsify(dec, 30)
    assert sdec.eta[3] == 0.0
    y = ranking.ObservationVector(12, k["iso_y_idx"], k["iso_y_val"], cap=3)
    h = ranking.h_alpha(0.99)
    xs = ranking.filter(sdec, h, y)
    np.testing.assert_allclose(xs, k["iso_x_sparse"], rtol=1e-9, atol=1e-12)
    assert xs[3] == 2.0
    # copy_uncovered=False leaves the zero score
    assert ranking.filter(sdec, h, y, copy_uncovered=False)[3] == 0.0


# ---------------------------------------------------------------- K7 -------
@pytest.mark.parametrize("dtype", ["float64", "float32"])
@pytest.mark.parametrize("tau", [1, 7, 500, 2999, 3000, 10 ** 9])
def test_sparsify_exact_tau_with_ties(dtype, tau):
    rng = np.random.default_rng(tau)
    U0 = rng.integers(-4, 5, size=(300, 10)).astype(np.float64) / 8.0  # heavy ties, exact zeros
    dt = N.torch_dtype(dtype)
    dec = spectral.SpectralDecomposition(torch.as_tensor(U0).to("cuda", dt), np.ones(10),
                                         torch.zeros(300, dtype=torch.float64, device="cuda"),
                                         None, spectral.Variant.APPROX, spectral.Provenance())
    sdec = spectral.sparsify(dec, tau)
    coo = sdec.U.tocoo()
    got = np.sort(coo.row.astype(np.int64) * 10 + coo.col)
    np.testing.assert_array_equal(got, O.sparsify_support(U0, tau))
    Ut, eta = O.sparsify(U0, tau)
    np.testing.assert_array_equal(sdec.U.toarray(), Ut.toarray())
    np.testing.assert_allclose(sdec.eta, eta, rtol=1e-12)


def test_sparsify_rejects():
    dec = spectral.SpectralDecomposition(torch.ones(3, 2, device="cuda", dtype=torch.float64), np.ones(2),
                                         torch.ones(3, dtype=torch.float64, device="cuda"), None,
                                         spectral.Variant.APPROX, spectral.Provenance())
    with pytest.raises(ValueError):
        spectral.sparsify(dec, 0)
    s = spectral.sparsify(dec, 2)
    with pytest.raises(ValueError):
        spectral.sparsify(s, 2)


# ------------------------------------------------------------ top-k --------
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_topk_matches_rank(dtype):
    rng = np.random.default_rng(5)
    b, n = 6, 50_000
    X = rng.standard_normal((b, n))
    X[1] = np.round(X[1], 1)           # many ties -> index order decides
    X[2] = 0.0                         # all ties
    X[2, [5, 70, 9000]] = [1.0, -2.0, 1.0]
    X[3, :n // 2] = -0.0
    dt = N.torch_dtype(dtype)
    Xd = torch.as_tensor(X).to("cuda", dt)
    Xr = Xd.double().cpu().numpy()
    K = 100
    idx = torch.empty(b, K, dtype=torch.int64, device="cuda")
    val = torch.empty(b, K, dtype=dt, device="cuda")
    N.Context.get().call("topk_rows", N.dtype_code(dt), b, n, N.ptr(Xd), n, K, N.ptr(idx), N.ptr(val))
    for j in range(b):
        np.testing.assert_array_equal(idx[j].cpu().numpy(), O.rank(Xr[j])[:K])


@pytest.mark.parametrize("b,n,K", [(1, 1_000_003, 100), (3, 200_000, 100), (7, 65_536, 1), (147, 70_001, 17),
                                   (2, 150_000, 1024)])
def test_topk_few_rows_histogram_path(b, n, K):
    """b < #SMs, n >= 65536, fp32: the two-pass histogram top-k (topk.cuh
    few_rows_*) equals the reference rank order and the segmented path's
    output bit for bit -- ties (rounded values, a row of zeros with more than
    kCap candidates -> the in-kernel exact fallback), -0.0, rows whose length
    is not a multiple of the vector width; the self-cleaning state survives
    repeated calls."""
    rng = np.random.default_rng(b * 1000 + K)
    X = rng.standard_normal((b, n)).astype(np.float32)
    X[0] = np.round(X[0], 1)
    if b > 1:
        X[1] = 0.0
        X[1, [5, 70, 9000]] = [1.0, -2.0, 1.0]
    if b > 2:
        X[2, : n // 2] = -0.0
        X[2, n // 2:] = np.abs(X[2, n // 2:]) * 1e-30  # one key bin holds half the row
    Xd = torch.as_tensor(X).cuda()
    ctx = N.Context.get()
    out = []
    for segs in (0, 0, 16):  # histogram path twice (state reuse), then the segmented path
        ctx.set_topk_segments(segs)
        idx = torch.empty(b, K, dtype=torch.int64, device="cuda")
        val = torch.empty(b, K, dtype=torch.float32, device="cuda")
        try:
            ctx.call("topk_rows", N.F32, b, n, N.ptr(Xd), n, K, N.ptr(idx), N.ptr(val))
        finally:
            ctx.set_topk_segments(0)
        out.append((idx.cpu().numpy(), val.cpu().numpy()))
    for j in range(b):
        order = O.rank(X[j].astype(np.float64))[:K]
        np.testing.assert_array_equal(out[0][0][j], order)
        np.testing.assert_array_equal(out[0][1][j].view(np.int32), X[j][order].view(np.int32))
    for o in out[1:]:
        np.testing.assert_array_equal(o[0], out[0][0])
        np.testing.assert_array_equal(o[1].view(np.int32), out[0][1].view(np.int32))


# ------------------------------------------------------- K9 at b = 1 -------
def _skewed_sparse_dec(n, r, seed):
    """Sparse U with skewed rows for the b = 1 SpMV (K9): empty rows, runs of
    empty rows, rows of 1 .. r entries around the 32/128-entry load widths."""
    from types import SimpleNamespace

    rng = np.random.default_rng(seed)
    lens = rng.choice([0, 1, 3, 31, 32, 33, 54, 255, 256, 257, 600], size=n,
                      p=[.15, .1, .1, .05, .05, .05, .3, .05, .05, .05, .05])
    lens[64:160] = 0                       # three empty groups
    lens[5] = r                            # a full row
    lens = np.minimum(lens, r)
    indptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    cols = np.concatenate([np.sort(rng.choice(r, size=k, replace=False)) for k in lens]).astype(np.int32)
    vals = rng.standard_normal(indptr[-1])
    U = sp.csr_matrix((vals, cols, indptr), shape=(n, r))
    eta = np.sqrt(np.asarray(U.multiply(U).sum(axis=1)).ravel())
    lam = np.sort(rng.uniform(-0.5, 1.0, r))[::-1].copy()
    return SimpleNamespace(U=U, eigenvalues=lam, eta=eta, variant="sparse", provenance=None, components=None)


@pytest.mark.parametrize("dtype,tol", [("float64", 1e-12), ("float32", 1e-5)])
def test_filter_b1_spmv_skewed_rows(dtype, tol):
    n, r = 3001, 700
    host = _skewed_sparse_dec(n, r, 11)
    dec = spectral.SpectralDecomposition.from_host(host, dtype=dtype)
    h = ranking.h_alpha(0.9)
    w = O.transfer_values(O.h_alpha(0.9), host.eigenvalues)
    for yi in ([5], [0, 7, 100, 2999], [64, 65]):
        y = ranking.ObservationVector(n, np.array(yi), np.linspace(1.0, 0.5, len(yi)), cap=len(yi))
        x = ranking.filter_batch(dec, h, [y])[0]
        ref = O.filter_scores(host.U, host.eigenvalues, host.eta, w, y.indices, y.values)
        err = np.linalg.norm(x - ref) / max(np.linalg.norm(ref), 1e-300)
        assert err <= tol, (yi, err)
        rows = np.flatnonzero(np.diff(host.U.indptr) == 0)
        np.testing.assert_array_equal(x[rows[~np.isin(rows, yi)]], 0.0)


def test_single_query_u16_columns_bitwise():
    """b = 1 fp32 filtering reads 16-bit column indices (fsr_filter_batch_u16):
    the same scores, bit for bit, as the int32-column kernel."""
    from paper_1703_06935_b200 import ranking

    rng = np.random.default_rng(23)
    n, r = 50_000, 700
    lens = rng.integers(0, 60, size=n)
    indptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    cols = np.concatenate([np.sort(rng.choice(r, size=k, replace=False)) for k in lens]).astype(np.int32)
    U = sp.csr_matrix((rng.standard_normal(indptr[-1]), cols, indptr), shape=(n, r))
    from types import SimpleNamespace

    eta = np.sqrt(np.asarray(U.multiply(U).sum(axis=1)).ravel())
    host = SimpleNamespace(U=U, eigenvalues=np.sort(rng.uniform(-0.3, 1, r))[::-1].copy(), eta=eta,
                           variant="sparse", provenance=None, components=None)
    dec = spectral.SpectralDecomposition.from_host(host, dtype="float32")
    y = ranking.ObservationVector(n, np.array([3, 999, 40_000]), np.array([1.0, 0.5, 0.2]), cap=3)
    q = ranking.DeviceQueries(ranking.QueryBatch.from_vectors([y]), dec.dtype, dec.eta_device.device)
    h = ranking.h_alpha(0.99)
    ctx = N.Context.get()
    ctx.single_query_path = "csr"  # the CSR SpMV with 16-bit columns (the default is K9e, below)
    try:
        x16 = ranking.filter_device(dec, h, q).X.clone()
    finally:
        ctx.single_query_path = "sell"
    Ud = dec.U_device
    w = ranking._weights_device(dec, h)
    ws = torch.empty(int(ctx.lib.fsr_filter_workspace_bytes(N.F32, n, r, 1, 1)), dtype=torch.uint8, device="cuda")
    x32 = torch.empty(1, n, dtype=torch.float32, device="cuda")
    ctx.call("filter_batch", N.F32, n, r, 1, N.ptr(Ud.indptr), N.ptr(Ud.indices), N.ptr(Ud.values), N.ptr(None), 0,
             N.ptr(w), N.ptr(dec.eta_device), 1, N.ptr(q.y_ptr), N.ptr(q.y_idx), N.ptr(q.y_val), 1, N.ptr(ws),
             N.ptr(x32), 0, N.ptr(None), N.ptr(None))
    torch.cuda.synchronize()
    assert torch.equal(x16.view(torch.int32), x32.view(torch.int32))


# ------------------------------------------- K9e: sliced-ELL single query ---
def _sequential_x(dec, h, y, n):
    """Row 0 of the unpruned wide-batch K9 (spmm_rowpanel_T_kernel: every x_i
    the sequential CSR-order fmaf chain) for a batch of 256 copies of y."""
    q = ranking.DeviceQueries(ranking.QueryBatch.from_vectors([y] * 256), dec.dtype, dec.eta_device.device)
    return ranking.filter_device(dec, h, q).X[0].clone()


@pytest.mark.parametrize("n,r,long_row", [(3001, 700, 512), (3001, 700, 40), (31, 64, 512), (4096, 300, 1),
                                          (50_000, 700, 512), (50_000, 700, None)])
def test_single_query_sell_bitwise_sequential(n, r, long_row, monkeypatch):
    """K9e (b = 1 on the sliced-ELL copy of U~) returns, bit for bit, the
    sequential-order sums of the wide-batch kernel: skewed rows, empty rows,
    rows on the CSR long-row path (long_row small: most rows; 1: every row),
    n not a multiple of 32, n < 32; top-k of the same call = exact rank order."""
    monkeypatch.setattr(ranking, "SELL_LONG_ROW", long_row)
    monkeypatch.setattr(ranking, "SELL_MAX_LONG_SHARE", 1.0)  # exercise the long-row path whatever its share
    host = _skewed_sparse_dec(n, r, 5) if n != 50_000 else _skewed_sparse_dec(n, r, 6)
    dec = spectral.SpectralDecomposition.from_host(host, dtype="float32")
    h = ranking.h_alpha(0.99)
    ctx = N.Context.get()
    assert ctx.single_query_path == "sell"
    lay = ranking.sell_layout(dec)
    assert lay is not None
    perm, lens, slice_ptr, cols, vals, n_long = lay
    rl = np.diff(host.U.indptr)
    np.testing.assert_array_equal(np.sort(perm.cpu().numpy()), np.arange(n))
    np.testing.assert_array_equal(lens.cpu().numpy(), rl[perm.cpu().numpy()])
    assert np.all(np.diff(lens.cpu().numpy()) <= 0) and n_long % 32 == 0
    if long_row is not None:  # None: the smallest candidate length within the long-share cap
        assert n_long >= np.count_nonzero(rl > long_row)
    for yi in ([5], [0, 7, min(100, n - 2), n - 1], [20, 21]):
        y = ranking.ObservationVector(n, np.array(yi), np.linspace(1.0, 0.5, len(yi)), cap=len(yi))
        q = ranking.DeviceQueries(ranking.QueryBatch.from_vectors([y]), dec.dtype, dec.eta_device.device)
        K = min(100, n)
        res = ranking.filter_device(dec, h, q, topk=K)
        seq = _sequential_x(dec, h, y, n)
        assert torch.equal(res.X[0].view(torch.int32), seq.view(torch.int32)), yi
        x = res.X[0].cpu().numpy()
        np.testing.assert_array_equal(res.top_idx[0].cpu().numpy(), O.rank(x)[:K])
        np.testing.assert_array_equal(res.top_val[0].cpu().numpy(), x[O.rank(x)[:K]])
        w = O.transfer_values(O.h_alpha(0.99), host.eigenvalues)
        ref = O.filter_scores(host.U, host.eigenvalues, host.eta, w, y.indices, y.values)
        assert np.linalg.norm(x - ref) <= 1e-5 * max(np.linalg.norm(ref), 1e-30)


@pytest.mark.parametrize("b", [2, 3, 4, 5, 8, 33, 64])
@pytest.mark.parametrize("n,r,long_row", [(3001, 700, 512), (3001, 700, 40), (50_000, 700, 512)])
def test_small_batch_sell_bitwise_sequential(b, n, r, long_row, monkeypatch):
    """K9e with 2 / 4 queries per pass (2 <= b <= 64): every row of X is, bit
    for bit, the sequential-order row of the wide-batch kernel, ragged last
    passes and empty queries included; the top-k is the reference rank order."""
    monkeypatch.setattr(ranking, "SELL_LONG_ROW", long_row)
    monkeypatch.setattr(ranking, "SELL_MAX_LONG_SHARE", 1.0)
    monkeypatch.setattr(ranking, "SELL_MAX_BATCH", 64)  # the library's limit (the host routes b <= 16 by default)
    host = _skewed_sparse_dec(n, r, 5)
    dec = spectral.SpectralDecomposition.from_host(host, dtype="float32")
    h = ranking.h_alpha(0.99)
    rng = np.random.default_rng(b)
    ys = []
    for j in range(b):
        k = 0 if j == 1 else int(rng.integers(1, 6))
        idx = np.sort(rng.choice(n, size=k, replace=False))
        ys.append(ranking.ObservationVector(n, idx, rng.uniform(0.1, 1.0, k), cap=max(k, 1)))
    dev = dec.eta_device.device
    q = ranking.DeviceQueries(ranking.QueryBatch.from_vectors(ys), dec.dtype, dev)
    K = 50
    res = ranking.filter_device(dec, h, q, topk=K)
    wide = ys + [ys[0]] * (256 - b)
    qw = ranking.DeviceQueries(ranking.QueryBatch.from_vectors(wide), dec.dtype, dev)
    seq = ranking.filter_device(dec, h, qw).X[:b]
    assert torch.equal(res.X.view(torch.int32), seq.view(torch.int32))
    X = res.X.cpu().numpy()
    for j in range(b):
        order = O.rank(X[j].astype(np.float64))[:K]
        np.testing.assert_array_equal(res.top_idx[j].cpu().numpy(), order)
        np.testing.assert_array_equal(res.top_val[j].cpu().numpy(), X[j][order])


def test_single_query_sell_policy_long_share(monkeypatch):
    """A U~ whose long rows hold more than SELL_MAX_LONG_SHARE of the entries
    keeps the CSR single-query kernel (sell_layout -> None); scores stay within
    the fp32 tolerance of the oracle."""
    monkeypatch.setattr(ranking, "SELL_LONG_ROW", 40)
    n, r = 3001, 700
    host = _skewed_sparse_dec(n, r, 5)
    dec = spectral.SpectralDecomposition.from_host(host, dtype="float32")
    assert ranking.sell_layout(dec) is None
    h = ranking.h_alpha(0.99)
    y = ranking.ObservationVector(n, np.array([0, 7, 100]), np.array([1.0, 0.5, 0.2]), cap=3)
    x = ranking.filter_batch(dec, h, [y])[0]
    w = O.transfer_values(O.h_alpha(0.99), host.eigenvalues)
    ref = O.filter_scores(host.U, host.eigenvalues, host.eta, w, y.indices, y.values)
    assert np.linalg.norm(x - ref) <= 1e-5 * np.linalg.norm(ref)


def test_single_query_sell_adaptive_long_row():
    """Default policy: the smallest candidate long-row length whose longer rows
    hold at most SELL_MAX_LONG_SHARE of the entries (none -> no layout)."""
    n, r = 50_000, 700
    host = _skewed_sparse_dec(n, r, 6)
    dec = spectral.SpectralDecomposition.from_host(host, dtype="float32")
    rl = np.diff(host.U.indptr)
    lay = ranking.sell_layout(dec)
    ok = [c for c in ranking.SELL_LONG_ROW_CANDIDATES
          if rl[rl > c].sum() <= ranking.SELL_MAX_LONG_SHARE * host.U.nnz]
    if not ok:
        assert lay is None
        return
    assert lay is not None
    n_long = lay[5]
    # every row over the chosen length sits in the long region, and the region holds whole slices
    assert n_long % 32 == 0 and n_long >= np.count_nonzero(rl > ok[0])
    assert n_long < np.count_nonzero(rl > ok[0]) + 32


def test_single_query_sell_graph_replay_and_csr_agree():
    """FilterGraph at b = 1 runs K9e; its top-100 equals the eager call's and the
    CSR single-query path's scores agree to rounding (another summation order)."""
    n, r = 50_000, 700
    host = _skewed_sparse_dec(n, r, 9)
    dec = spectral.SpectralDecomposition.from_host(host, dtype="float32")
    h = ranking.h_alpha(0.9)
    y = ranking.ObservationVector(n, np.array([3, 999, 40_000]), np.array([1.0, 0.5, 0.2]), cap=3)
    qb = ranking.QueryBatch.from_vectors([y])
    q = ranking.DeviceQueries(qb, dec.dtype, dec.eta_device.device)
    eager = ranking.filter_device(dec, h, q, topk=100)
    fg = ranking.FilterGraph(dec, h, b=1, nnz_cap=8, topk=100)
    res = fg.run(qb)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(res.top_idx[0].cpu().numpy(), eager.top_idx[0].cpu().numpy())
    np.testing.assert_array_equal(res.top_val[0].cpu().numpy(), eager.top_val[0].cpu().numpy())
    ctx = N.Context.get()
    ctx.single_query_path = "csr"
    try:
        xc = ranking.filter_device(dec, h, q).X[0].cpu().numpy()
    finally:
        ctx.single_query_path = "sell"
    xs = eager.X[0].cpu().numpy()
    assert np.linalg.norm(xc - xs) <= 2e-6 * np.linalg.norm(xs)
