"""Certified pruned top-k (csrc/prune.cuh): fp16-gathered K9 + exact fp32
re-score must return exactly the unpruned fp32 path's top-k -- the same
indices and bitwise the same values -- including ties, empty observations,
copied uncovered rows and queries that overflow the candidate buffer (the
device fallback)."""

from types import SimpleNamespace

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import fsr_oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1703_06935_b200 import _native as N  # noqa: E402
from paper_1703_06935_b200 import ranking, spectral  # noqa: E402


def make_dec(n, r, per_row, seed, dup_block=0, empty_every=0):
    rng = np.random.default_rng(seed)
    lens = rng.integers(max(1, per_row // 4), 2 * per_row, size=n)
    if empty_every:
        lens[::empty_every] = 0
    indptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    cols = np.concatenate([np.sort(rng.choice(r, size=k, replace=False)) for k in lens]).astype(np.int32)
    vals = rng.standard_normal(indptr[-1]) * rng.choice([1.0, 1e-3], size=indptr[-1], p=[0.9, 0.1])
    U = sp.csr_matrix((vals, cols, indptr), shape=(n, r))
    if dup_block:
        # dup_block copies of row 1 (identical scores -> ties broken by index)
        rows = [U[i] if not (1000 <= i < 1000 + dup_block) else U[1] for i in range(n)]
        U = sp.vstack(rows).tocsr()
    eta = np.sqrt(np.asarray(U.multiply(U).sum(axis=1)).ravel())
    lam = np.sort(rng.uniform(-0.3, 1.0, r))[::-1].copy()
    host = SimpleNamespace(U=U, eigenvalues=lam, eta=eta, variant="sparse", provenance=None, components=None)
    return host, spectral.SpectralDecomposition.from_host(host, dtype="float32")


def queries(n, b, seed, k=50, empty=(), extra=None):
    rng = np.random.default_rng(seed)
    ys = []
    for j in range(b):
        if j in empty:
            idx = np.array([], dtype=np.int64)
        else:
            idx = np.unique(rng.integers(0, n, size=k))
            if extra and j in extra:
                idx = np.unique(np.concatenate([idx, extra[j]]))
        ys.append(ranking.ObservationVector(n, idx, rng.random(idx.size) ** 3 + 0.01, cap=max(idx.size, 1)))
    return ranking.QueryBatch.from_vectors(ys)


# the certified paths under test: K9t (tensor cores, csrc/k9t.cu), K9s (packed
# fp16 U~ streamed from HBM, csrc/k9t.cu) and K9h (fp16 gathers, csrc/prune.cuh)
PATHS = ["tc", "stream", "pruned"]


@pytest.fixture(params=PATHS)
def path(request):
    ctx = N.Context.get()
    old = ctx.online_path
    ctx.set_online_path(request.param)
    yield request.param
    ctx.set_online_path(old)


def both(dec, qb, K=100, h=None, flags=None):
    """(certified path top-k, unpruned fp32 path top-k) of the same batch."""
    h = h or ranking.h_alpha(0.99)
    ctx = N.Context.get()
    dq = ranking.DeviceQueries(qb, dec.dtype, dec.eta_device.device)
    ws = torch.empty(ranking.filter_workspace_bytes(dec, qb.b, want_x=False, topk=K), dtype=torch.uint8,
                     device=dec.eta_device.device)
    assert ranking.online_path(dec, qb.b, K) == ctx.online_path
    out = []
    for prune in (True, False):
        ctx.set_topk_prune(prune)
        try:
            r = ranking.filter_device(dec, h, dq, topk=K, want_x=False, workspace=ws)
            torch.cuda.synchronize()
            out.append((r.top_idx.cpu().numpy(), r.top_val.cpu().numpy()))
            if prune:
                assert ctx.last_online_path == ctx.online_path
                if flags is not None:
                    flags.append(ranking.last_fallback_count(ws, dec, qb.b))
        finally:
            ctx.set_topk_prune(True)
    return out


@pytest.mark.parametrize("seed", [0, 1])
def test_pruned_topk_identical_to_unpruned(seed, path):
    n, r, b = 150_000, 600, 256
    host, dec = make_dec(n, r, 40, seed)
    qb = queries(n, b, seed + 10)
    fl = []
    (pi, pv), (ui, uv) = both(dec, qb, flags=fl)
    assert fl == [0]  # no query needed the fallback
    np.testing.assert_array_equal(pi, ui)
    np.testing.assert_array_equal(pv.view(np.uint32), uv.view(np.uint32))
    # and the unpruned fp32 path against the fp64 oracle on a few queries
    w = O.transfer_values(O.h_alpha(0.99), host.eigenvalues)
    for j in (0, 77, 255):
        idx = qb.y_idx[qb.y_ptr[j]:qb.y_ptr[j + 1]]
        val = qb.y_val[qb.y_ptr[j]:qb.y_ptr[j + 1]]
        x = O.filter_scores(host.U, host.eigenvalues, host.eta, w, idx, val)
        assert len(np.intersect1d(O.rank(x)[:100], pi[j])) >= 99
        np.testing.assert_allclose(pv[j], x[pi[j]], rtol=1e-4, atol=1e-5 * np.abs(x).max())


def test_pruned_ties_empty_uncovered_and_fallback(path):
    n, r, b = 140_000, 400, 256
    # 5000 identical rows overflow the candidate buffer for queries that hit row 1;
    # every 97th row is empty (uncovered when observed)
    host, dec = make_dec(n, r, 30, 3, dup_block=5000, empty_every=97)
    extra = {5: np.array([1]), 6: np.array([1, 97 * 3]), 9: np.array([97 * 5, 97 * 8])}
    qb = queries(n, b, 4, empty=(2, 200), extra=extra)
    fl = []
    (pi, pv), (ui, uv) = both(dec, qb, flags=fl)
    # K9h: the two empty observations and the queries on the duplicated rows;
    # K9t / K9s answer empty observations directly (k9t_empty), not by the fallback
    assert fl[0] >= (4 if path == "pruned" else 2)
    np.testing.assert_array_equal(pi, ui)
    np.testing.assert_array_equal(pv.view(np.uint32), uv.view(np.uint32))
    # empty observation: all-zero scores, first K indices
    np.testing.assert_array_equal(pi[2], np.arange(100))
    # copied uncovered rows carry y
    j = 9
    yv = dict(zip(qb.y_idx[qb.y_ptr[j]:qb.y_ptr[j + 1]], qb.y_val[qb.y_ptr[j]:qb.y_ptr[j + 1]]))
    for i in (97 * 5, 97 * 8):
        if i in pi[j]:
            assert pv[j][list(pi[j]).index(i)] == np.float32(yv[i])


def test_pruned_heat_kernel_k_range_ragged_batch(path):
    n, r, b = 131_072 + 5, 300, 264  # n not a multiple of 4, b not a multiple of the 256-column panel
    _, dec = make_dec(n, r, 20, 8)
    qb = queries(n, b, 9, k=30)
    for K, h in ((1, ranking.heat_kernel(10.0)), (37, ranking.h_alpha(0.9)), (128, ranking.h_alpha(0.99)), (256, ranking.h_alpha(0.99))):
        (pi, pv), (ui, uv) = both(dec, qb, K=K, h=h)
        np.testing.assert_array_equal(pi, ui)
        np.testing.assert_array_equal(pv.view(np.uint32), uv.view(np.uint32))


def test_filter_graph_partial_batch_on_pruned_path(path):
    """A CUDA-graph step over a partial batch (the padding queries are empty
    observations) returns the unpruned fp32 top-k for the real queries."""
    n, r, b = 140_000, 300, 256
    _, dec = make_dec(n, r, 20, 21)
    qb = queries(n, 100, 22)
    h = ranking.h_alpha(0.99)
    fg = ranking.FilterGraph(dec, h, b=b, nnz_cap=int(qb.y_ptr[-1]), topk=50)
    fg.submit(qb)
    gi, gv = fg.fetch()
    ctx = N.Context.get()
    ctx.set_topk_prune(False)
    try:
        r_ = ranking.filter_device(dec, h, ranking.DeviceQueries(qb, dec.dtype, dec.eta_device.device), topk=50,
                                   want_x=False)
        torch.cuda.synchronize()
    finally:
        ctx.set_topk_prune(True)
    np.testing.assert_array_equal(gi, r_.top_idx.cpu().numpy())
    np.testing.assert_array_equal(gv.view(np.uint32), r_.top_val.cpu().numpy().view(np.uint32))


def test_pruned_nonfinite_projection_matches_unpruned(path):
    """A query whose projection overflows fp32 (y values of 1e300 -> inf in the
    fp32 batch) has no finite bound: the pruned path must hand it to the exact
    fallback and return what the unpruned path returns (a NaN
    bound used to sort above +inf and pick wrong rows)."""
    n, r, b = 140_000, 300, 256
    _, dec = make_dec(n, r, 20, 31)
    qb = queries(n, b, 32)
    y_val = qb.y_val.copy()
    for j in (3, 70):
        s, e = qb.y_ptr[j], qb.y_ptr[j + 1]
        y_val[s:s + 3] = 1e300
    qb = ranking.QueryBatch(n, qb.y_ptr, qb.y_idx, y_val)
    fl = []
    (pi, pv), (ui, uv) = both(dec, qb, flags=fl)
    assert fl[0] >= 2
    np.testing.assert_array_equal(pi, ui)
    np.testing.assert_array_equal(pv.view(np.uint32), uv.view(np.uint32))
    ok = [j for j in range(b) if j not in (3, 70)]
    assert np.isfinite(pv[ok]).all()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs in one process")
def test_two_devices_one_process():
    """Kernel shared-memory attributes are per device: the pruned
    step (64 KB fallback select, large-smem K8) runs on a second device of the
    same process after the first."""
    n, r, b = 140_000, 300, 256
    host, _ = make_dec(n, r, 20, 41)
    qb = queries(n, b, 42)
    res = []
    for d in (0, 1):
        with torch.cuda.device(d):
            dec = spectral.SpectralDecomposition.from_host(host, dtype="float32", device=torch.device("cuda", d))
            dq = ranking.DeviceQueries(qb, dec.dtype, torch.device("cuda", d))
            r_ = ranking.filter_device(dec, ranking.h_alpha(0.99), dq, topk=100, want_x=False)
            torch.cuda.synchronize(d)
            res.append((r_.top_idx.cpu().numpy(), r_.top_val.cpu().numpy()))
    np.testing.assert_array_equal(res[0][0], res[1][0])
    np.testing.assert_array_equal(res[0][1].view(np.uint32), res[1][1].view(np.uint32))


@pytest.mark.parametrize("b", [1, 7, 64, 100, 200])
def test_tc_small_and_odd_batches(b, monkeypatch):
    """K9t at batch widths below its default minimum (forced), on each query
    tile width (64: b <= 64, 128: b <= 128, else 256) and not a multiple of
    it: same top-k as the unpruned path."""
    monkeypatch.setattr(ranking, "TC_MIN_BATCH", 1)
    monkeypatch.setattr(ranking, "tc_pays", lambda dec, b: True)  # force K9t below its cost-model crossover
    n, r = 70_001, 257
    _, dec = make_dec(n, r, 25, 51)
    qb = queries(n, b, 52, empty=(0,) if b > 2 else ())
    ctx = N.Context.get()
    old = ctx.online_path
    ctx.set_online_path("tc")
    try:
        (pi, pv), _ = both(dec, qb, K=100)
    finally:
        ctx.set_online_path(old)
    # the unpruned reference in the sequential per-row order: the same queries
    # padded with empty ones to a 256-wide batch (b <= 64 would take the narrow
    # exact kernels, which sum a row in interleaved halves)
    pad = ranking.QueryBatch(n, np.concatenate([qb.y_ptr, np.full(256 - b, qb.y_ptr[-1])]), qb.y_idx, qb.y_val)
    ctx.set_topk_prune(False)
    try:
        r_ = ranking.filter_device(dec, ranking.h_alpha(0.99), ranking.DeviceQueries(pad, dec.dtype,
                                   dec.eta_device.device), topk=100, want_x=False)
        torch.cuda.synchronize()
    finally:
        ctx.set_topk_prune(True)
    np.testing.assert_array_equal(pi, r_.top_idx[:b].cpu().numpy())
    np.testing.assert_array_equal(pv.view(np.uint32), r_.top_val[:b].cpu().numpy().view(np.uint32))


def padded_unpruned(dec, qb, K, h=None):
    """The unpruned reference in the sequential per-row order: the queries
    padded with empty ones to a 256-wide batch (b <= 64 would take the narrow
    exact kernels, which sum a row in interleaved halves)."""
    n, b = dec.n, qb.b
    pad = ranking.QueryBatch(n, np.concatenate([qb.y_ptr, np.full(256 - b, qb.y_ptr[-1])]), qb.y_idx, qb.y_val)
    ctx = N.Context.get()
    ctx.set_topk_prune(False)
    try:
        r_ = ranking.filter_device(dec, h or ranking.h_alpha(0.99), ranking.DeviceQueries(pad, dec.dtype,
                                   dec.eta_device.device), topk=K, want_x=False)
        torch.cuda.synchronize()
    finally:
        ctx.set_topk_prune(True)
    return r_.top_idx[:b].cpu().numpy(), r_.top_val[:b].cpu().numpy()


@pytest.mark.parametrize("b", [1, 2, 5, 8, 64, 100])
def test_stream_small_batches(b):
    """K9s (preferred) on small batches: one NB-query group per 8 queries,
    ragged last group; the sequential-order unpruned top-k bit for bit, also
    through a FilterGraph replay."""
    n, r = 140_003, 300
    _, dec = make_dec(n, r, 25, 61)
    qb = queries(n, b, 62, empty=(1,) if b > 4 else ())
    ctx = N.Context.get()
    tc = b >= ranking.TC_MIN_BATCH and ranking.tc_pays(dec, b)
    assert ranking.online_path(dec, b, 100) == ("tc" if tc else "exact")
    ctx.set_online_path("stream")
    try:
        _stream_small_batch_checks(dec, qb, b)
    finally:
        ctx.set_online_path("tc")


def _stream_small_batch_checks(dec, qb, b):
    ctx = N.Context.get()
    assert ranking.online_path(dec, b, 100) == "stream"
    dq = ranking.DeviceQueries(qb, dec.dtype, dec.eta_device.device)
    ws = torch.empty(ranking.filter_workspace_bytes(dec, b, want_x=False, topk=100), dtype=torch.uint8,
                     device=dec.eta_device.device)
    res = ranking.filter_device(dec, ranking.h_alpha(0.99), dq, topk=100, want_x=False, workspace=ws)
    torch.cuda.synchronize()
    assert ctx.last_online_path == "stream"
    assert ranking.last_fallback_count(ws, dec, b) == 0
    si, sv = res.top_idx.cpu().numpy(), res.top_val.cpu().numpy()
    ui, uv = padded_unpruned(dec, qb, 100)
    np.testing.assert_array_equal(si, ui)
    np.testing.assert_array_equal(sv.view(np.uint32), uv.view(np.uint32))
    fg = ranking.FilterGraph(dec, ranking.h_alpha(0.99), b=b, nnz_cap=int(qb.y_ptr[-1]), topk=100)
    fg.submit(qb)
    gi, gv = fg.fetch()
    np.testing.assert_array_equal(gi, ui)
    np.testing.assert_array_equal(gv.view(np.uint32), uv.view(np.uint32))


def test_stream_long_rows_tiny_and_empty_chunks():
    """Packed-stream chunking edge cases: rows as long as r (a chunk spans up
    to kChunk - 1 + r entries), runs of thousands of empty rows (chunks that
    hold many rows or none), and a U~ smaller than one chunk."""
    rng = np.random.default_rng(71)
    for n, r, full_rows in ((131_072, 512, 40), (3_000, 64, 2)):
        lens = rng.integers(0, 30, size=n)
        lens[rng.choice(n, full_rows, replace=False)] = r
        lens[5000:9000 if n > 9000 else 0] = 0
        if n < 5000:
            lens[:] = rng.integers(0, 2, size=n)  # nnz < one chunk
            lens[7] = r
        indptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        cols = np.concatenate([np.sort(rng.choice(r, size=k, replace=False)) for k in lens]).astype(np.int32)
        U = sp.csr_matrix((rng.standard_normal(indptr[-1]), cols, indptr), shape=(n, r))
        eta = np.sqrt(np.asarray(U.multiply(U).sum(axis=1)).ravel())
        lam = np.sort(rng.uniform(-0.3, 1.0, r))[::-1].copy()
        host = SimpleNamespace(U=U, eigenvalues=lam, eta=eta, variant="sparse", provenance=None, components=None)
        dec = spectral.SpectralDecomposition.from_host(host, dtype="float32")
        K = min(100, n)
        for b in (1, 8, 13):
            qb = queries(n, b, 72 + b, k=20)
            ctx = N.Context.get()
            ctx.set_online_path("stream")
            try:
                assert ranking.online_path(dec, b, K) == "stream"
                res = ranking.filter_device(dec, ranking.h_alpha(0.99), ranking.DeviceQueries(qb, dec.dtype,
                                            dec.eta_device.device), topk=K, want_x=False)
                torch.cuda.synchronize()
            finally:
                ctx.set_online_path("tc")
            ui, uv = padded_unpruned(dec, qb, K)
            np.testing.assert_array_equal(res.top_idx.cpu().numpy(), ui)
            np.testing.assert_array_equal(res.top_val.cpu().numpy().view(np.uint32), uv.view(np.uint32))
