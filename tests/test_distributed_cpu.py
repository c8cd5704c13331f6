"""Row-sharded offline FSR with world_size 2 on the gloo backend (CPU).

The orchestration of paper_1703_06935_b200.distributed (collectives, offsets,
tie ordering across ranks) is driven with numpy local ops and compared with
the single-process oracle: Ritz values, U (same sign rule), eta and the exact
sparse support.
"""

import os
import socket

import numpy as np
import pytest
import scipy.sparse as sp
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import fsr_oracle as O


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def problem(n=240, seed=3):
    rng = np.random.default_rng(seed)
    M = rng.random((n, n)) * (rng.random((n, n)) < 0.05)
    M = np.triu(M, 1)
    M[5, :] = 0.0
    M[:, 5] = 0.0
    W = sp.csr_matrix(M + M.T)
    return O.normalize_adjacency(W, O.degrees(W))


def worker(rank, world, port, out_path, r, p, q, tau, ties):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1703_06935_b200 import _native as N
        from paper_1703_06935_b200 import distributed as D
        from dist_numpy_ops import NumpyOps

        S = problem()
        comm = D.Comm()
        shard = D.make_shard(comm, S.indptr)
        A_local = S[shard.r0:shard.r1]
        ops = NumpyOps()
        stats = []
        Q, B = D.sharded_range_finder(comm, ops, A_local, shard, r + p, q, 0, N.F64, stats)
        U, lam, eta = D.sharded_rayleigh_ritz(comm, ops, Q, B, r, shard)
        Uh = U.numpy().copy()
        if ties:
            Uh = np.round(Uh * 8) / 8  # force many ties across the rank boundary
            U = torch.as_tensor(Uh)
        Ut, eta_s, keep = D.sharded_sparsify(comm, ops, U, tau, shard, N.F64)
        coo = Ut.tocoo()
        flat = (coo.row.astype(np.int64) + shard.r0) * r + coo.col
        np.savez(f"{out_path}.{rank}.npz", U=Uh, lam=lam, eta=eta.numpy(), flat=flat, eta_s=eta_s,
                 r0=shard.r0, keep=keep, stats=np.array(stats))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("ties,world", [(False, 2), (True, 2), (False, 4)])
def test_sharded_matches_oracle(tmp_path, ties, world):
    r, p, q, tau = 12, 6, 3, 700
    out = str(tmp_path / "res")
    mp.spawn(worker, args=(world, free_port(), out, r, p, q, tau, ties), nprocs=world, join=True)
    parts = [np.load(f"{out}.{k}.npz") for k in range(world)]
    S = problem()
    U_ref, lam_ref, eta_ref = O.decompose(S, r, p=p, q=q, seed=0)
    lam = parts[0]["lam"]
    for pt in parts[1:]:
        np.testing.assert_array_equal(lam, pt["lam"])  # redundant eigh: identical on all ranks
    assert np.abs(lam - lam_ref).max() <= 1e-10 * np.abs(lam_ref).max()
    U = np.concatenate([pt["U"] for pt in parts])
    if ties:
        U_ref = np.round(U_ref * 8) / 8
    else:
        assert np.abs(U - U_ref).max() < 1e-8
        np.testing.assert_allclose(np.concatenate([pt["eta"] for pt in parts]), eta_ref, atol=1e-10)
    flat = np.sort(np.concatenate([pt["flat"] for pt in parts]))
    np.testing.assert_array_equal(flat, O.sparsify_support(U, tau))
    assert parts[0]["keep"] == min(tau, np.count_nonzero(U))


def test_row_partition_balances_nnz():
    from paper_1703_06935_b200.distributed import row_partition

    indptr = np.concatenate([[0], np.cumsum(np.arange(100) % 7)])
    parts = row_partition(indptr, 4)
    assert parts[0][0] == 0 and parts[-1][1] == 100
    assert all(a <= b for a, b in parts)
    loads = [indptr[b] - indptr[a] for a, b in parts]
    assert max(loads) - min(loads) <= 12
    assert row_partition(np.zeros(1, np.int64), 3) == [(0, 0)] * 3


def pipeline_worker(rank, world, port, out_path, panel):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1703_06935_b200 import _native as N
        from paper_1703_06935_b200 import distributed as D
        from dist_numpy_ops import NumpyOps

        D.EXCHANGE_PANEL = panel
        S = problem()
        comm = D.Comm()
        shard = D.make_shard(comm, S.indptr)
        ops = NumpyOps()
        Q, B = D.sharded_range_finder(comm, ops, S[shard.r0:shard.r1], shard, 18, 3, 0, N.F64)
        # the collectives themselves: rank-ordered sum, ragged (and empty) row shards
        rng = np.random.default_rng(100 + rank)
        part = torch.as_tensor(rng.standard_normal((7, 5)))
        tot = comm.sum_ordered(part)
        counts = [3, 0, 5, 1][:world] if world <= 4 else [2] * world
        mine = torch.full((counts[rank], 2), float(rank))
        rows = comm.all_gather_rows(mine, counts)
        np.savez(f"{out_path}.{rank}.npz", Q=Q.numpy(), B=B.numpy(), part=part.numpy(), tot=tot.numpy(),
                 rows=rows.numpy(), counts=np.array(counts))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_panel_pipelined_exchange_is_bitwise_unpipelined(tmp_path, world):
    """exchange_spmm in 5-column panels (ragged last panel, two buffers in
    flight) gives bitwise the Q and B of the whole-block exchange; sum_ordered
    (all-to-all + rank-ordered adds + all-gather) equals ((p0 + p1) + p2) + ...
    bit for bit on every rank; all_gather_rows handles ragged and empty shards."""
    res = {}
    for panel in (5, 0):
        out = str(tmp_path / f"p{panel}")
        mp.spawn(pipeline_worker, args=(world, free_port(), out, panel), nprocs=world, join=True)
        res[panel] = [np.load(f"{out}.{k}.npz") for k in range(world)]
    for k in range(world):
        np.testing.assert_array_equal(res[5][k]["Q"], res[0][k]["Q"])
        np.testing.assert_array_equal(res[5][k]["B"], res[0][k]["B"])
    parts = [res[5][k]["part"] for k in range(world)]
    acc = parts[0].copy()
    for p in parts[1:]:
        acc += p
    counts = res[5][0]["counts"]
    want_rows = np.concatenate([np.full((c, 2), float(k)) for k, c in enumerate(counts)])
    for k in range(world):
        np.testing.assert_array_equal(res[5][k]["tot"], acc)
        np.testing.assert_array_equal(res[5][k]["rows"], want_rows)
