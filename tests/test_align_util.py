"""The comparison helper itself (CPU): cluster_align recovers per-window signs and
within-cluster rotations, and never mixes columns across step windows."""
import numpy as np

from tests._util import cluster_align


def test_cluster_align_recovers_rotations_and_signs():
    rng = np.random.default_rng(0)
    n, b = 12, 4
    ur = np.linalg.qr(rng.standard_normal((20, n)))[0]
    d = np.array([3, 2, 2, 2, 1.5, 1, .5, .4, .3, .3, .1, .05])
    r = np.eye(n)
    r[1:4, 1:4] = np.linalg.qr(rng.standard_normal((3, 3)))[0]
    r[8:10, 8:10] = np.linalg.qr(rng.standard_normal((2, 2)))[0]
    s = np.diag(rng.choice([-1.0, 1.0], n))
    ug = ur @ r @ s
    D = cluster_align(ug, ur, d, b)
    assert np.max(np.abs(ur @ D - ug)) < 1e-14
    assert np.allclose(D.T @ D, np.eye(n))


def test_cluster_align_is_window_local():
    # equal values straddling a window boundary are NOT merged: only signs there
    n, b = 8, 4
    d = np.array([4.0, 3.0, 1.0, 1.0, 1.0, 1.0, 0.5, 0.2])
    u = np.eye(n)
    D = cluster_align(u, u, d, b)
    assert np.allclose(D, np.eye(n))
    assert np.count_nonzero(D[:4, 4:]) == 0 and np.count_nonzero(D[4:, :4]) == 0
