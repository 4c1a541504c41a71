"""Near-equal singular values inside one step's window (config 4's sigma = 1 block):
the B200 result matches the oracle after the within-window Procrustes alignment of
SURVEY.md section 8a.2 (tests/_util.cluster_align), with the reference's own G."""
import numpy as np
import pytest

import oracle
import paper_2104_05782_b200 as rutv
from tests._util import check_structure, cluster_align, residual

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,b,q,k", [(256, 32, 2, 80), (300, 64, 1, 100), (200, 48, 2, 30)])
def test_cliff_cluster_matches_oracle_after_alignment(n, b, q, k):
    i = np.arange(1, n + 1)
    sig = np.where(i <= k, 1.0, 1e-3 * 0.999 ** (i - k))
    a = oracle.spectrum_matrix(n, n, sig, 11)
    g = oracle.normal_stream(4, 0, oracle.stream_length(n, n, b))
    t, u, v = rutv.factorize(a, b=b, q=q, seed=4, g=g)
    tr, ur, vr = oracle.randutv(a, b=b, q=q, seed=4)
    check_structure(t, b)
    assert residual(a, t, u, v) < 1e-13
    D = cluster_align(u, ur, np.diag(tr), b, rel=1e-8)
    nf = np.linalg.norm(a)
    du = np.max(np.abs(u - ur @ D))
    dv = np.max(np.abs(v - vr @ D))
    dt = np.max(np.abs(t - D.T @ tr @ D)) / nf
    dd = np.max(np.abs(np.diag(t) - np.diag(tr)))
    # the cluster diagonal (sigma = 1) is invariant under the alignment
    assert dd <= 1e-12, dd
    assert du <= 1e-9 and dv <= 1e-9 and dt <= 1e-11, (du, dv, dt)
