"""Near-equal singular values (config 4's sigma = 1 block) against the oracle, with the
reference's own G.

SURVEY.md section 8a.2: inside a cluster of (near-)equal singular values the Jacobi
SVD of a step's b x b window fixes the basis only up to a rounding-determined
rotation.  Windows that lie entirely inside the cluster are therefore compared
after the within-window Procrustes alignment (tests/_util.cluster_align): U, V,
T rows there must agree to rounding.  The window that straddles the cliff mixes
the cluster with whichever tail directions the sketch captured; those diagonal
entries are sensitive to rounding in the REFERENCE ITSELF (a 1.1e-16 relative
perturbation of A moves them by up to ~5e-6 at n = 256), so the diagonal is held
to 1000 x the reference's own sensitivity, measured here on the same input.
"""
import numpy as np
import pytest

import oracle
import paper_2104_05782_b200 as rutv
from tests._util import check_structure, cluster_align, residual

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,b,q,k", [(256, 32, 2, 80), (300, 64, 1, 100), (200, 24, 2, 60)])
def test_cliff_cluster_matches_oracle_after_alignment(n, b, q, k):
    i = np.arange(1, n + 1)
    sig = np.where(i <= k, 1.0, 1e-3 * 0.999 ** (i - k))
    a = oracle.spectrum_matrix(n, n, sig, 11)
    g = oracle.normal_stream(4, 0, oracle.stream_length(n, n, b))
    t, u, v = rutv.factorize(a, b=b, q=q, seed=4, g=g)
    tr, ur, vr = oracle.randutv(a, b=b, q=q, seed=4)
    check_structure(t, b)
    assert residual(a, t, u, v) < 1e-13
    # the reference's own rounding sensitivity on this input
    rng = np.random.default_rng(1)
    selfd = np.zeros(n)
    for _ in range(2):
        ap = np.asfortranarray(a * (1 + 1.1e-16 * rng.standard_normal(a.shape)))
        selfd = np.maximum(selfd, np.abs(np.diag(oracle.randutv(ap, b=b, q=q, seed=4)[0]) - np.diag(tr)))
    dd = np.abs(np.diag(t) - np.diag(tr))
    assert np.all(dd <= 1e3 * selfd + 1e-14), (np.argmax(dd - 1e3 * selfd), dd.max(), selfd.max())
    c = (k // b) * b  # windows entirely inside the sigma = 1 cluster
    D = cluster_align(u, ur, np.diag(tr), b, rel=1e-8)
    nf = np.linalg.norm(a)
    du = np.max(np.abs(u - ur @ D)[:, :c])
    dv = np.max(np.abs(v - vr @ D)[:, :c])
    dt = np.max(np.abs(t - D.T @ tr @ D)[:c, :c]) / nf
    assert np.max(np.abs(np.diag(t)[:c] - 1.0)) <= 1e-13
    assert du <= 1e-12 and dv <= 1e-12 and dt <= 1e-13, (du, dv, dt)
