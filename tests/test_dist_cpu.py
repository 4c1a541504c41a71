"""Multi-rank gloo tests of the multi-GPU schedule (paper_2104_05782_b200/dist.py) on CPU.

The distributed driver runs with the CPU test double (tests/_dist_ops.py:
reference-convention QR and Jacobi from the oracle, torch fp64 GEMMs), P x Q
processes over gloo on 127.0.0.1; the gathered T, U, V must match the
single-process oracle randutv (proj/src/randutv_blocked.cpp:84-157) after the
SVD sign alignment of SURVEY.md 8a.2.  Grids 1x2, 2x1, 2x2, 1x3 and 2x3 cover
the row communicator, the column communicator, both, odd counts and ragged
tails.  Also covers the block-cyclic index math against the reference's
formula (proj/src/block_cyclic.cpp:26-38).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import oracle
from paper_2104_05782_b200.dist import Grid, Layout, grid_shape


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, P, Q, port, n, b, q, seed_a, seed_g, use_g, out_path):
    import torch.distributed as dist
    from paper_2104_05782_b200.dist import factorize_dist, gather_grid, scatter_grid
    from tests._dist_ops import TorchCpuOps
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=P * Q)
    try:
        torch.set_num_threads(1)
        grid = Grid(n, b, P, Q, rank)
        a = torch.from_numpy(oracle.gaussian_matrix(n, n, seed_a).T.copy()).T
        a_loc = scatter_grid(a, grid)
        g = None
        if use_g:
            g = torch.from_numpy(oracle.normal_stream(seed_g, 0, oracle.stream_length(n, n, b)))
        t, u, v = factorize_dist(a_loc, grid, q=q, seed=seed_g, ops=TorchCpuOps(), g=g)
        T, U, V = gather_grid(t, grid), gather_grid(u, grid), gather_grid(v, grid)
        if rank == 0:
            np.savez(out_path, t=T.numpy(), u=U.numpy(), v=V.numpy())
    finally:
        dist.destroy_process_group()


def _run_and_check(tmp_path, P, Q, n, b, q, seed_a=11, seed_g=5, use_g=False):
    out = str(tmp_path / "res.npz")
    mp.spawn(_worker, args=(P, Q, _free_port(), n, b, q, seed_a, seed_g, use_g, out), nprocs=P * Q, join=True)
    r = np.load(out)
    a = oracle.gaussian_matrix(n, n, seed_a)
    tr, ur, vr = oracle.randutv(a, b=b, q=q, seed=seed_g)
    d = np.sign(np.einsum("ij,ij->j", r["u"], ur))
    d[d == 0] = 1
    nf = np.linalg.norm(a)
    assert np.max(np.abs(r["t"] - d[:, None] * tr * d[None, :])) / nf < 1e-12
    assert np.max(np.abs(r["u"] - ur * d)) < 1e-10
    assert np.max(np.abs(r["v"] - vr * d)) < 1e-10
    assert np.all(np.tril(r["t"], -1) == 0.0)
    assert np.linalg.norm(a - r["u"] @ r["t"] @ r["v"].T) / nf < 1e-13


@pytest.mark.parametrize("n,b,q", [(64, 16, 1), (70, 16, 2), (100, 32, 0), (97, 8, 1)])
def test_1x2_grid_matches_oracle(tmp_path, n, b, q):
    _run_and_check(tmp_path, 1, 2, n, b, q)


@pytest.mark.parametrize("n,b,q", [(64, 16, 1), (75, 16, 2)])
def test_2x1_grid_matches_oracle(tmp_path, n, b, q):
    _run_and_check(tmp_path, 2, 1, n, b, q)


@pytest.mark.parametrize("n,b,q,use_g", [(96, 16, 1, False), (90, 16, 2, True), (53, 8, 0, False)])
def test_2x2_grid_matches_oracle(tmp_path, n, b, q, use_g):
    _run_and_check(tmp_path, 2, 2, n, b, q, seed_a=3, seed_g=9, use_g=use_g)


def test_1x3_ragged(tmp_path):
    _run_and_check(tmp_path, 1, 3, 90, 16, 1, seed_a=3, seed_g=9, use_g=True)


def test_2x3_ragged(tmp_path):
    _run_and_check(tmp_path, 2, 3, 101, 8, 1, seed_a=4, seed_g=6)


def test_grid_matches_reference_block_cyclic_formula():
    # block_cyclic.cpp:26-38: owner(br, bc) = (br mod P) Q + (bc mod Q), local (br div P, bc div Q)
    for n, b, P, Q in [(100, 16, 1, 2), (97, 8, 1, 3), (4000, 128, 2, 4), (50000, 512, 2, 4), (30000, 256, 2, 2),
                       (101, 8, 2, 3)]:
        seen = {}
        for rank in range(P * Q):
            gr = Grid(n, b, P, Q, rank)
            for kr in gr.rows.owned():
                for kc in gr.cols.owned():
                    assert gr.owner2(kr, kc) == rank
                    assert gr.rows.loc(kr) == b * (kr // P)
                    assert gr.cols.loc(kc) == b * (kc // Q)
                    seen[(kr, kc)] = rank
            mr, mc = gr.local_shape()
            assert mr == sum(gr.width(k) for k in gr.rows.owned())
            assert mc == sum(gr.width(k) for k in gr.cols.owned())
        nb = Grid(n, b, P, Q, 0).nblk
        assert len(seen) == nb * nb
        assert sum(np.prod(Grid(n, b, P, Q, r).local_shape()) for r in range(P * Q)) == n * n
    for world, pq in [(1, (1, 1)), (2, (1, 2)), (4, (2, 2)), (8, (2, 4)), (6, (2, 3))]:
        assert grid_shape(world) == pq


def test_layout_is_the_1xQ_grid():
    for n, b, world in [(100, 16, 2), (97, 8, 3), (4000, 128, 8)]:
        seen = []
        for rank in range(world):
            lay = Layout(n, b, world, rank)
            for k in lay.owned():
                assert lay.owner(k) == k % world == rank == lay.owner2(0, k)
                assert lay.loc_off(k) == sum(lay.width(j) for j in lay.owned() if j < k)
            seen += lay.owned()
            assert lay.local_shape() == (n, lay.ncols())
        assert sorted(seen) == list(range(Layout(n, b, world, 0).nblk))
