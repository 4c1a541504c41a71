"""The distributed driver's GPU ops (dist.CudaOps + NCCL) on one B200 (world size 1).

Multi-rank NCCL cannot run on the single GPU the test box offers; the
multi-rank schedule is covered by tests/test_dist_cpu.py (gloo, 2 and 3 ranks).
Here the same driver runs with our kernels through the asynchronous C ABI and
NCCL collectives, and must agree with the oracle like the single-GPU path.
"""
import os
import socket

import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture(scope="module")
def nccl_group():
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_port())
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
    yield
    dist.destroy_process_group()


@pytest.mark.parametrize("n,b,q,use_g", [(200, 32, 1, True), (256, 64, 2, True), (300, 128, 0, False), (193, 64, 1, True)])
def test_dist_cudaops_world1_matches_oracle(nccl_group, n, b, q, use_g):
    from paper_2104_05782_b200.dist import CudaOps, Layout, factorize_dist, scatter_columns
    from tests._util import cm_cuda, to_np
    a = oracle.gaussian_matrix(n, n, 21)
    lay = Layout(n, b, 1, 0)
    a_loc = scatter_columns(cm_cuda(a), lay)
    g = torch.from_numpy(oracle.normal_stream(4, 0, oracle.stream_length(n, n, b))).cuda() if use_g else None
    t, u, v = factorize_dist(a_loc, lay, q=q, seed=4, ops=CudaOps(torch.device("cuda:0")), g=g)
    tg, ug, vg = to_np(t), to_np(u), to_np(v)
    tr, ur, vr = oracle.randutv(a, b=b, q=q, seed=4)
    d = np.sign(np.einsum("ij,ij->j", ug, ur))
    d[d == 0] = 1
    nf = np.linalg.norm(a)
    tol_t = 1e-11 if use_g else 1e-10
    assert np.max(np.abs(tg - d[:, None] * tr * d[None, :])) / nf < tol_t
    dg, dr = np.diag(tg), np.diag(tr)
    assert np.max(np.abs(dg - dr) / np.abs(dr)) < 1e-9
    # U/V entries of the trailing, nearly degenerate singular directions are
    # rounding-sensitive; invariants pin them instead.
    assert np.max(np.abs(ug - ur * d)) < 1e-7 and np.max(np.abs(vg - vr * d)) < 1e-7
    assert np.linalg.norm(a - ug @ tg @ vg.T) / nf < 1e-13
    assert np.linalg.norm(ug.T @ ug - np.eye(n)) < 1e-12 and np.linalg.norm(vg.T @ vg - np.eye(n)) < 1e-12
    assert np.all(np.tril(tg, -1) == 0.0)
