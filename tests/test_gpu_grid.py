"""The sharded 2D block-cyclic factorization (dist.cu) on the B200.

The box has one GPU, so the P x Q ranks run as host threads on it with the in-process
exchange (grid_sim): the SAME driver code as the NCCL path, only the collectives
differ (device copies behind host barriers; no kernel ever waits on another rank's
kernel).  Checked against the oracle with the reference's own G, on grids from 1 x 2
to 3 x 2, ragged n, ranks that run out of blocks, and no-U/V; the NCCL backend itself
runs at world size 1 through the multi-process entry points.
"""
import numpy as np
import pytest
import torch

import oracle
import paper_2104_05782_b200 as rutv
from tests._util import check_structure, compare_to_oracle, orth_defect, residual

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,b,q,grid", [(300, 64, 1, (1, 2)), (300, 64, 1, (2, 1)), (256, 32, 2, (2, 2)),
                                        (333, 48, 1, (2, 3)), (200, 32, 0, (3, 2)), (130, 16, 2, (1, 3)),
                                        (520, 128, 2, (2, 2)), (100, 32, 1, (2, 4))])
def test_grid_matches_oracle(n, b, q, grid):
    a = oracle.gaussian_matrix(n, n, 77 + n)
    g = oracle.normal_stream(3, 0, oracle.stream_length(n, n, b))
    got = rutv.factorize(a, b=b, q=q, seed=3, g=g, grid=grid, grid_sim=True)
    ref = oracle.randutv(a, b=b, q=q, seed=3)
    t, u, v = got
    check_structure(t, b)
    assert residual(a, t, u, v) < 1e-13
    assert orth_defect(u) < 1e-12 and orth_defect(v) < 1e-12
    # The pure-relative diag test is held to the reference's OWN rounding sensitivity on this
    # input (q = 2 amplifies rounding in the smallest diagonal entries: a 1.1e-16 relative
    # perturbation of A moves them by up to ~1e-10 relative at n = 520), floor 1e-10.
    ap = np.asfortranarray(a * (1 + 1.1e-16 * np.random.default_rng(1).standard_normal(a.shape)))
    dself = np.max(np.abs(np.diag(oracle.randutv(ap, b=b, q=q, seed=3)[0]) - np.diag(ref[0])) / np.abs(np.diag(ref[0])))
    compare_to_oracle(a, got, ref, diag_rel=max(1e-10, 10 * dself))


def test_grid_matches_single_gpu_device_rng():
    n, b, q = 400, 64, 1
    a = oracle.gaussian_matrix(n, n, 5)
    t1, u1, v1 = rutv.factorize(a, b=b, q=q, seed=9)
    t2, u2, v2 = rutv.factorize(a, b=b, q=q, seed=9, grid=(2, 2), grid_sim=True)
    # each rank draws its own rows of G from the counter stream: same deviates as one GPU
    d = np.sign(np.einsum("ij,ij->j", u2, u1))
    assert np.max(np.abs(np.diag(t2) - np.diag(t1)) / np.diag(t1)) < 1e-10
    assert np.max(np.abs(u2 - u1 * d)) < 1e-9 and np.max(np.abs(v2 - v1 * d)) < 1e-9


def test_grid_tall_panels_match_single_gpu():
    """n above RUTV_CHOLQR_MIN_ROWS (4608): every rank factors the gathered sketch and the
    diagonal owner the panel through the Cholesky-QR2 sub-panels, each reading its safety flag
    back with a host synchronisation of its own critical stream -- inside the rank threads of
    the in-process grid.  Device RNG on both sides; max_steps bounds the run."""
    n, b, q, steps = 6656, 256, 1, 3
    a = torch.empty((n, n), dtype=torch.float64, device="cuda").T
    rutv.gaussian_matrix_device(a, 11)
    ah = np.asfortranarray(a.cpu().numpy())
    t1, u1, v1 = rutv.factorize(ah, b=b, q=q, seed=9, max_steps=steps)
    t2, u2, v2 = rutv.factorize(ah, b=b, q=q, seed=9, max_steps=steps, grid=(1, 2), grid_sim=True)
    k = steps * b
    d = np.sign(np.einsum("ij,ij->j", u2[:, :k], u1[:, :k]))
    assert np.max(np.abs(np.diag(t2)[:k] - np.diag(t1)[:k]) / np.diag(t1)[:k]) < 1e-10
    assert np.max(np.abs(u2[:, :k] - u1[:, :k] * d)) < 1e-9 and np.max(np.abs(v2[:, :k] - v1[:, :k] * d)) < 1e-9
    nf = np.linalg.norm(ah)
    assert np.linalg.norm(ah - u2 @ t2 @ v2.T) / nf < 1e-13


def test_grid_no_uv_same_t():
    n, b, q = 260, 32, 1
    a = oracle.gaussian_matrix(n, n, 8)
    g = oracle.normal_stream(1, 0, oracle.stream_length(n, n, b))
    t1, _, _ = rutv.factorize(a, b=b, q=q, seed=1, g=g, grid=(2, 2), grid_sim=True)
    t2, u2, v2 = rutv.factorize(a, b=b, q=q, seed=1, g=g, grid=(2, 2), grid_sim=True, build_uv=False)
    assert u2 is None and v2 is None
    assert np.array_equal(t1, t2)


def test_grid_is_deterministic():
    n, b, q = 300, 48, 2
    a = oracle.gaussian_matrix(n, n, 2)
    r1 = rutv.factorize(a, b=b, q=q, seed=4, grid=(2, 3), grid_sim=True)
    r2 = rutv.factorize(a, b=b, q=q, seed=4, grid=(2, 3), grid_sim=True)
    for x, y in zip(r1, r2):
        assert np.array_equal(x, y)


def test_grid_errors():
    a = oracle.gaussian_matrix(30, 20, 1)
    with pytest.raises(rutv.RutvError):  # the sharded path is square-only
        rutv.factorize(a, b=8, q=1, grid=(1, 2), grid_sim=True)
    sq = oracle.gaussian_matrix(40, 40, 1)
    with pytest.raises(ValueError):  # needs P*Q GPUs without grid_sim
        rutv.factorize(sq, b=8, q=1, grid=(4, 4))


def test_nccl_world1_multiprocess_entry():
    """rutv_b200_nccl_unique_id / dist_create / factorize_dist over a real NCCL communicator
    (world 1 on the one-GPU box), local blocks == the whole matrix, stacked [V; T] in place."""
    n, b, q = 384, 64, 1
    a = oracle.gaussian_matrix(n, n, 6)
    g = oracle.normal_stream(2, 0, oracle.stream_length(n, n, b))
    ref = rutv.factorize(a, b=b, q=q, seed=2, g=g)
    ctx = rutv.DistContext(rutv.nccl_unique_id(), 1, 1, 0, 0)
    mr, mc = rutv.grid_local_shape(n, b, 1, 1, 0)
    assert (mr, mc) == (n, n)
    full = torch.from_numpy(np.ascontiguousarray(a.T)).cuda().T
    a_loc = torch.empty((mc, mr), dtype=torch.float64, device="cuda").T
    rutv.grid_copy(full, a_loc, n, b, 1, 1, 0, to_local=True)
    vt = torch.empty((mc, 2 * mr), dtype=torch.float64, device="cuda").T
    u = torch.empty((mc, mr), dtype=torch.float64, device="cuda").T
    ctx.factorize(n, a_loc, vt[mr:, :], u, vt[:mr, :], b=b, q=q, seed=2, g=torch.from_numpy(g).cuda())
    ctx.close()
    got = (vt[mr:, :].cpu().numpy(), u.cpu().numpy(), vt[:mr, :].cpu().numpy())
    compare_to_oracle(a, got, ref, t_tol=1e-12, uv_tol=1e-10, diag_rel=1e-11)
