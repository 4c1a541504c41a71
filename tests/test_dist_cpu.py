"""World-size-2 gloo tests of the multi-GPU schedule (paper_2104_05782_b200/dist.py) on CPU.

The distributed driver runs with the CPU test double (tests/_dist_ops.py:
reference-convention QR and Jacobi from the oracle, torch fp64 GEMMs), two
processes over gloo on 127.0.0.1; the gathered T, U, V must match the
single-process oracle randutv (proj/src/randutv_blocked.cpp:84-157) after the
SVD sign alignment of SURVEY.md 8a.2.  Also covers the block-cyclic index math
against the reference's formula (proj/src/block_cyclic.cpp:26-38).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import oracle
from paper_2104_05782_b200.dist import Layout


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, n, b, q, seed_a, seed_g, use_g, out_path):
    import torch.distributed as dist
    from paper_2104_05782_b200.dist import factorize_dist, gather_columns, scatter_columns
    from tests._dist_ops import TorchCpuOps
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.set_num_threads(1)
        lay = Layout(n, b, world, rank)
        a = torch.from_numpy(oracle.gaussian_matrix(n, n, seed_a).T.copy()).T
        a_loc = scatter_columns(a, lay)
        g = None
        if use_g:
            g = torch.from_numpy(oracle.normal_stream(seed_g, 0, oracle.stream_length(n, n, b)))
        t, u, v = factorize_dist(a_loc, lay, q=q, seed=seed_g, ops=TorchCpuOps(), g=g)
        T = gather_columns(t, lay, n)
        U = gather_columns(u, lay, n)
        V = gather_columns(v, lay, n)
        if rank == 0:
            np.savez(out_path, t=T.numpy(), u=U.numpy(), v=V.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("n,b,q", [(64, 16, 1), (70, 16, 2), (100, 32, 0), (97, 8, 1)])
def test_two_rank_schedule_matches_oracle(tmp_path, n, b, q):
    out = str(tmp_path / "res.npz")
    mp.spawn(_worker, args=(2, _free_port(), n, b, q, 11, 5, False, out), nprocs=2, join=True)
    r = np.load(out)
    a = oracle.gaussian_matrix(n, n, 11)
    tr, ur, vr = oracle.randutv(a, b=b, q=q, seed=5)
    d = np.sign(np.einsum("ij,ij->j", r["u"], ur))
    d[d == 0] = 1
    nf = np.linalg.norm(a)
    assert np.max(np.abs(r["t"] - d[:, None] * tr * d[None, :])) / nf < 1e-12
    assert np.max(np.abs(r["u"] - ur * d)) < 1e-10
    assert np.max(np.abs(r["v"] - vr * d)) < 1e-10
    assert np.all(np.tril(r["t"], -1) == 0.0)
    assert np.linalg.norm(a - r["u"] @ r["t"] @ r["v"].T) / nf < 1e-13


def test_three_rank_ragged(tmp_path):
    n, b, q = 90, 16, 1
    out = str(tmp_path / "res.npz")
    mp.spawn(_worker, args=(3, _free_port(), n, b, q, 3, 9, True, out), nprocs=3, join=True)
    r = np.load(out)
    a = oracle.gaussian_matrix(n, n, 3)
    tr, ur, vr = oracle.randutv(a, b=b, q=q, seed=9)
    d = np.sign(np.einsum("ij,ij->j", r["u"], ur))
    d[d == 0] = 1
    assert np.max(np.abs(r["t"] - d[:, None] * tr * d[None, :])) / np.linalg.norm(a) < 1e-12


def test_layout_matches_reference_block_cyclic_formula():
    # block_cyclic.cpp:26-38 with a 1 x Q grid: owner = bc mod Q, local index = bc div Q
    for n, b, world in [(100, 16, 2), (97, 8, 3), (4000, 128, 8), (50000, 512, 8)]:
        seen = []
        for rank in range(world):
            lay = Layout(n, b, world, rank)
            for k in lay.owned():
                assert lay.owner(k) == k % world == rank
                assert lay.loc_off(k) == sum(lay.width(j) for j in lay.owned() if j < k)
            seen += lay.owned()
            assert lay.ncols() == sum(lay.width(k) for k in lay.owned())
        assert sorted(seen) == list(range(Layout(n, b, world, 0).nblk))
        assert sum(Layout(n, b, world, r).ncols() for r in range(world)) == n
