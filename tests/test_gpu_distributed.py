"""Sharded offline path on the GPU: world_size 1 in-process, and 2 ranks on
one GPU over gloo (host-staged collectives; no kernel waits on another rank).
Checked against the C1 golden fixtures of the reference."""

import hashlib
import os
import socket

import numpy as np
import pytest
import scipy.sparse as sp

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "c1.npz")


def c1():
    g = dict(np.load(GOLD))
    n, r, p, q, tau, seed = (int(v) for v in g["params"])
    S = sp.csr_matrix((g["S_data"], g["W_indices"], g["W_indptr"]), shape=(n, n))
    return g, S, (n, r, p, q, tau, seed)


def run(comm_world, rank, out, dtype="float64"):
    from paper_1703_06935_b200 import distributed as D

    g, S, (n, r, p, q, tau, seed) = c1()
    comm = D.Comm()
    res = D.sharded_decompose(comm, S, r, p, q, seed, tau=tau, dtype=dtype, device="cuda:0")
    sh = res["shard"]
    Ut = res["Ut"].to_scipy().tocoo()
    flat = (Ut.row.astype(np.int64) + sh.r0) * r + Ut.col
    full = D.gather_csr(comm, res["Ut"], sh)
    np.savez(out, lam=res["eigenvalues"], flat=flat, eta=res["eta"].cpu().numpy(), r0=sh.r0,
             full_nnz=full.nnz, full_rows=full.to_scipy().getnnz(axis=1))


def worker(rank, world, port, out, dtype="float64"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        run(world, rank, f"{out}.{rank}.npz", dtype)
    finally:
        dist.destroy_process_group()


def check(parts, g, r, dtype="float64"):
    lam = parts[0]["lam"]
    if dtype == "float32":  # fast mode: Ritz normwise 1e-5; sparsify keeps exactly tau entries
        assert np.abs(lam - g["lam"]).max() <= 1e-5 * np.abs(g["lam"]).max()
        eta = np.concatenate([pt["eta"] for pt in parts])
        assert np.abs(eta - g["eta"]).max() < 1e-4
        for pt in parts:
            assert int(pt["full_nnz"]) == int(g["sparse_nnz"])
        return
    assert np.abs(lam - g["lam"]).max() <= 1e-10 * np.abs(g["lam"]).max()
    flat = np.sort(np.concatenate([pt["flat"] for pt in parts]))
    assert hashlib.sha256(flat.astype(np.int64).tobytes()).hexdigest() == str(g["sparse_hash"])
    eta = np.concatenate([pt["eta"] for pt in parts])
    assert np.abs(eta - g["eta"]).max() < 1e-8
    for pt in parts:
        assert int(pt["full_nnz"]) == int(g["sparse_nnz"])


def test_sharded_world1(tmp_path):
    g, _, (n, r, *_rest) = c1()
    out = str(tmp_path / "w1.npz")
    run(1, 0, out)
    check([np.load(out)], g, r)


@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_sharded_two_ranks_one_gpu(tmp_path, dtype):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    out = str(tmp_path / "w2")
    mp.spawn(worker, args=(2, port, out, dtype), nprocs=2, join=True)
    g, _, (n, r, *_rest) = c1()
    parts = [np.load(f"{out}.{k}.npz") for k in range(2)]
    np.testing.assert_array_equal(parts[0]["lam"], parts[1]["lam"])
    check(parts, g, r, dtype)
