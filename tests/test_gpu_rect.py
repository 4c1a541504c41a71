"""Rectangular m x n and qr_prepass on the B200 against the oracle.

Shapes follow test_randutv_blocked.cpp:81-96 (30x20, 20x30, 13x7, the
1x7 / 7x1 degenerate ones, :187-207) and the qr_prepass case (:173-185), plus
larger tall / wide inputs whose last step takes the rectangular dense SVD
with orthonormal completion (jacobi_svd.cpp:150-240)."""
import numpy as np
import pytest

import oracle
import paper_2104_05782_b200 as rutv
from tests._util import check_structure

pytestmark = pytest.mark.gpu


def _col_signs(x, y):
    d = np.sign(np.einsum("ij,ij->j", x, y))
    d[d == 0] = 1.0
    return d


def _invariants(a, t, u, v, b):
    m, n = a.shape
    assert t.shape == (m, n) and u.shape == (m, m) and v.shape == (n, n)
    nf = max(np.linalg.norm(a), 1e-300)
    assert np.linalg.norm(a - u @ t @ v.T) / nf < 1e-12
    assert np.linalg.norm(u.T @ u - np.eye(m)) < 1e-11
    assert np.linalg.norm(v.T @ v - np.eye(n)) < 1e-11
    check_structure(t, b)
    if min(m, n) > 0:
        sa = np.linalg.svd(a, compute_uv=False)
        st = np.linalg.svd(t, compute_uv=False)
        assert np.max(np.abs(sa - st)) < 1e-11 * max(sa[0], 1e-300)


def _parity(a, got, ref, t_tol=1e-11, uv_tol=1e-8):
    """Sign-aligned parity.  For wide inputs (m < n) the trailing n - m columns
    of V span null(A); the reference fixes them through Householder vectors of
    a rank-deficient sketch, i.e. by rounding noise, so only the
    first m columns are compared entrywise (the rest is then the same subspace)."""
    tg, ug, vg = got
    tr, ur, vr = ref
    m, n = a.shape
    du, dv = _col_signs(ug, ur), _col_signs(vg, vr)
    nf = max(np.linalg.norm(a), 1e-300)
    assert np.max(np.abs(tg - du[:, None] * tr * dv[None, :])) / nf < t_tol
    assert np.max(np.abs(ug - ur * du[None, :])) < uv_tol
    k = min(m, n)
    assert np.max(np.abs(vg[:, :k] - vr[:, :k] * dv[None, :k]), initial=0.0) < uv_tol


@pytest.mark.parametrize("m,n,b,q", [(30, 20, 8, 0), (20, 30, 8, 2), (13, 7, 5, 1), (24, 24, 8, 1),
                                     (1, 7, 4, 1), (7, 1, 4, 1), (300, 200, 32, 1), (200, 300, 32, 2),
                                     (700, 300, 64, 1), (300, 700, 64, 1), (129, 257, 64, 1),
                                     (513, 100, 128, 0), (100, 513, 128, 1)])
def test_rectangular_matches_oracle(m, n, b, q):
    a = oracle.gaussian_matrix(m, n, 300 + 31 * m + n)
    g = oracle.normal_stream(7, 0, max(oracle.stream_length(m, n, b), 1))
    got = rutv.factorize(a, b=b, q=q, seed=7, g=g)
    ref = oracle.randutv(a, b=b, q=q, seed=7)
    _invariants(a, *got, b)
    _parity(a, got, ref)


@pytest.mark.parametrize("m,n,b,q", [(40, 10, 4, 1), (600, 100, 32, 1), (2000, 300, 128, 2)])
def test_qr_prepass_matches_oracle(m, n, b, q):
    a = oracle.gaussian_matrix(m, n, 340 + m)
    g = oracle.normal_stream(9, 0, oracle.stream_length(n, n, b))
    got = rutv.factorize(a, b=b, q=q, seed=9, g=g, qr_prepass=True)
    ref = oracle.randutv(a, b=b, q=q, seed=9, qr_prepass=True)
    _invariants(a, *got, b)
    assert np.all(got[0][n:, :] == 0.0)  # rows below the square part are exact zeros
    _parity(a, got, ref)


def test_rectangular_device_rng_and_no_uv():
    m, n, b = 500, 260, 64
    a = oracle.gaussian_matrix(m, n, 77)
    t, u, v = rutv.factorize(a, b=b, q=1, seed=3)
    _invariants(a, t, u, v, b)
    t2, u2, v2 = rutv.factorize(a, b=b, q=1, seed=3, build_uv=False)
    assert u2 is None and v2 is None
    assert np.array_equal(t, t2)


def test_rank_deficient_tall_completion():
    # rank-2 tall input: the final dense block is rank deficient, so U's
    # completion takes over most columns
    rng = np.random.default_rng(5)
    a = rng.standard_normal((90, 2)) @ rng.standard_normal((2, 20))
    g = oracle.normal_stream(4, 0, oracle.stream_length(90, 20, 8))
    got = rutv.factorize(a, b=8, q=1, seed=4, g=g)
    ref = oracle.randutv(a, b=8, q=1, seed=4)
    _invariants(a, *got, 8)
    tg, tr = got[0], ref[0]
    assert np.max(np.abs(np.abs(tg) - np.abs(tr))) < 1e-10 * np.linalg.norm(a)
