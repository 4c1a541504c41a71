"""Kernel-level parity of the sm_100a kernels against the CPU oracle.

Mirrors the reference's kernel tests: gemm (test_matrix.cpp:143-189),
Householder (test_householder.cpp:33-200), Jacobi (test_block_svd.cpp:86-238),
RNG (test_matrix.cpp:222-278).  All calls go through the C ABI.
"""
import numpy as np
import pytest

import oracle
import paper_2104_05782_b200 as rutv
from tests._util import cm_cuda, cm_empty, orth_defect, to_np

pytestmark = pytest.mark.gpu


def _rand(m, n, seed):
    return oracle.gaussian_matrix(m, n, seed)


# ------------------------------------------------------------------ GEMM --
GEMM_SHAPES = [
    # (M, N, K) -- the step catalogue of SURVEY.md 8a at small s, plus ragged edges
    (5, 3, 4), (64, 64, 64), (130, 127, 129), (500, 128, 500), (128, 372, 500),
    (1000, 128, 1000), (128, 128, 2000), (2000, 2000, 128), (777, 33, 65), (1, 1, 1),
]


@pytest.mark.parametrize("ta", [0, 1])
@pytest.mark.parametrize("tb", [0, 1])
@pytest.mark.parametrize("shape", GEMM_SHAPES)
def test_gemm_matches_oracle(shape, ta, tb):
    M, N, K = shape
    a = _rand(*((K, M) if ta else (M, K)), 11)
    b = _rand(*((N, K) if tb else (K, N)), 12)
    c0 = _rand(M, N, 10)
    for alpha, beta in [(1.0, 0.0), (-0.75, 1.0), (1.0, 0.5)]:
        c = cm_cuda(c0)
        rutv.gemm(alpha, ta, cm_cuda(a), tb, cm_cuda(b), beta, c)
        want = oracle.gemm(alpha, ta, a, tb, b, beta, c0)
        err = np.max(np.abs(to_np(c) - want))
        scale = np.sqrt(K) * 8.0
        assert err < 1e-13 * scale, (shape, ta, tb, alpha, beta, err)


def test_gemm_beta_zero_overwrites_nan():
    a, b = _rand(70, 40, 2), _rand(40, 50, 3)
    c = cm_empty(70, 50, fill=float("nan"))
    rutv.gemm(1.0, 0, cm_cuda(a), 0, cm_cuda(b), 0.0, c)
    assert np.all(np.isfinite(to_np(c)))


def test_gemm_unaligned_views():
    # odd offsets / leading dims take the 8-byte cp.async path
    big = _rand(301, 211, 5)
    import torch
    A = cm_cuda(big)
    av = A[3:3 + 97, 1:1 + 65]       # odd row offset -> unaligned
    bv = A[1:1 + 65, 7:7 + 33]
    c = cm_empty(97, 33)
    rutv.gemm(1.0, 0, av, 0, bv, 0.0, c)
    want = big[3:100, 1:66] @ big[1:66, 7:40]
    assert np.max(np.abs(to_np(c) - want)) < 1e-12
    assert torch.cuda.is_available()


def test_gemm_shape_error():
    with pytest.raises(ValueError):
        rutv.gemm(1.0, 0, cm_empty(3, 4), 0, cm_empty(5, 2), 0.0, cm_empty(3, 2))


def test_gemm_deterministic():
    a, b = _rand(3000, 128, 21), _rand(3000, 128, 22)
    outs = []
    for _ in range(3):
        c = cm_empty(128, 128)
        rutv.gemm(1.0, 1, cm_cuda(a), 0, cm_cuda(b), 0.0, c)
        outs.append(to_np(c))
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[1], outs[2])


# ------------------------------------------------------------------- RNG --
def test_normal_fill_matches_host_stream():
    import torch
    rows, cols, pos = 1000, 37, 123457
    g = cm_empty(rows, cols)
    rutv.normal_fill(42, pos, g)
    host = oracle.normal_stream(42, pos, rows * cols).reshape(cols, rows).T
    dev = to_np(g)
    diff = np.abs(dev - host)
    # integer layer is exact; libm differences are ulp-level only
    assert np.max(diff / np.maximum(np.abs(host), 1.0)) < 1e-14
    exact = np.mean(dev == host)
    assert exact > 0.5, f"only {exact:.3f} of deviates bit-identical"
    assert torch.cuda.is_available()


# ----------------------------------------------------------- Householder --
@pytest.mark.parametrize("m,n", [(8, 5), (5, 5), (9, 2), (200, 16), (1000, 128), (4000, 128),
                                 (3000, 256), (50, 64), (37, 40), (300, 17), (513, 33), (2000, 128),
                                 (10000, 64), (20000, 24)])
def test_hqr_matches_oracle(m, n):
    a = _rand(m, n, 100 + m)
    qr_ref, tau_ref, twy_ref = oracle.hqr(a)
    p = min(m, n)
    import torch
    A = cm_cuda(a)
    tau = torch.zeros(p, dtype=torch.float64, device="cuda")
    twy = cm_empty(p, p)
    rutv.hqr(A, tau, twy)
    qr = to_np(A)
    assert np.all(np.diag(qr)[:p] >= 0.0)
    scale = np.linalg.norm(a)
    assert np.max(np.abs(np.triu(qr)[:p] - np.triu(qr_ref)[:p])) < 1e-12 * scale
    assert np.max(np.abs(np.tril(qr, -1) - np.tril(qr_ref, -1))) < 1e-10
    assert np.max(np.abs(tau.cpu().numpy() - tau_ref)) < 1e-12
    assert np.max(np.abs(to_np(twy) - twy_ref)) < 1e-10


def test_hqr_reference_edge_conventions():
    import torch
    # already-triangular: tau = 0 and the input is returned bit-equal (test_householder.cpp:114-121)
    a = np.zeros((4, 4))
    for j in range(4):
        for i in range(j + 1):
            a[i, j] = 1 + i + j
    A = cm_cuda(a)
    tau = torch.zeros(4, dtype=torch.float64, device="cuda")
    rutv.hqr(A, tau, cm_empty(4, 4))
    assert np.all(tau.cpu().numpy() == 0.0)
    assert np.array_equal(to_np(A), a)
    # negative head, no tail: tau = 2, R = +2 (test_householder.cpp:123-130)
    a = np.eye(3)
    a[0, 0] = -2.0
    A = cm_cuda(a)
    tau = torch.zeros(3, dtype=torch.float64, device="cuda")
    rutv.hqr(A, tau, cm_empty(3, 3))
    assert to_np(A)[0, 0] == 2.0 and tau.cpu().numpy()[0] == 2.0


@pytest.mark.parametrize("s,p,rows", [(8, 4, 5), (500, 64, 300), (2000, 128, 4000)])
def test_apply_q_matches_oracle(s, p, rows):
    a = _rand(s, p, 60)
    qr, tau, twy = oracle.hqr(a)
    bmat = _rand(rows, s, 61)
    want = oracle.apply_q_right(qr, twy, bmat)
    B = cm_cuda(bmat)
    rutv.apply_q_right(cm_cuda(qr), cm_cuda(twy), B)
    assert np.max(np.abs(to_np(B) - want)) < 1e-12 * np.sqrt(s)
    bl = _rand(s, rows, 62)
    want = oracle.apply_qt_left(qr, twy, bl)
    B = cm_cuda(bl)
    rutv.apply_qt_left(cm_cuda(qr), cm_cuda(twy), B)
    assert np.max(np.abs(to_np(B) - want)) < 1e-12 * np.sqrt(s)


# ---------------------------------------------------------------- Jacobi --
def _svd_dev(a, **kw):
    import torch
    n = a.shape[0]
    U, V = cm_empty(n, n), cm_empty(n, n)
    s = torch.zeros(max(n, 1), dtype=torch.float64, device="cuda")
    rutv.svd_block(cm_cuda(a), U, s, V, **kw)
    return to_np(U), s.cpu().numpy()[:n], to_np(V)


@pytest.mark.parametrize("n", [1, 2, 5, 16, 63, 128, 129, 256, 336, 512])
def test_svd_block_reconstructs(n):
    a = _rand(n, n, 200 + n)
    u, s, v = _svd_dev(a)
    assert orth_defect(u) < 1e-12 * max(1, n / 16) and orth_defect(v) < 1e-12 * max(1, n / 16)
    assert np.all(s[:-1] >= s[1:]) and np.all(s >= 0)
    rec = (u * s) @ v.T
    assert np.max(np.abs(rec - a)) < 1e-12 * (1 + np.linalg.norm(a))
    _, s_ref, _ = oracle.svd_block(a)
    assert np.max(np.abs(s - s_ref)) < 1e-13 * max(s_ref[0], 1.0) * max(1, n / 16)


def test_svd_block_known_answer_2x2():
    # jacobi test_block_svd.cpp:131-141: sigma = sqrt(45), sqrt(5)
    a = np.array([[3.0, 0.0], [4.0, 5.0]])
    _, s, _ = _svd_dev(a)
    assert abs(s[0] - np.sqrt(45.0)) < 1e-14 * np.sqrt(45) and abs(s[1] - np.sqrt(5.0)) < 1e-14 * 3


def test_svd_block_zero_and_rank_one():
    u, s, v = _svd_dev(np.zeros((3, 3)))
    assert np.all(s == 0) and orth_defect(u) < 1e-14 and orth_defect(v) < 1e-14
    x, y = _rand(5, 1, 220), _rand(5, 1, 221)
    a = x @ y.T
    u, s, v = _svd_dev(a)
    want = np.linalg.norm(x) * np.linalg.norm(y)
    assert abs(s[0] - want) < 1e-12 * want and np.all(s[1:] < 1e-12 * want)
    assert orth_defect(u) < 1e-11 and orth_defect(v) < 1e-11


def test_svd_block_sweep_cap():
    with pytest.raises(rutv.ConvergenceError) as ei:
        _svd_dev(_rand(6, 6, 230), max_sweeps=0)
    assert ei.value.residual > 0.0


def test_svd_block_geometric_diagonal():
    n = 12
    a = np.diag(0.5 ** np.arange(n))
    _, s, _ = _svd_dev(a)
    assert np.max(np.abs(s - 0.5 ** np.arange(n)) / 0.5 ** np.arange(n)) < 1e-13


def test_twy_with_identity_reflectors():
    """Twy when some tau = 0 (householder.cpp:26-27: H = I): form_t's inverse form
    does not exist there and the kernel takes the recurrence (householder.cpp:76-97)."""
    import torch
    s, p = 300, 40
    a = oracle.gaussian_matrix(s, p, 17)
    for j in (0, 1, 2):  # leading columns already upper triangular, positive diagonal -> tau_j = 0
        a[j + 1:, j] = 0.0
        a[j, j] = abs(a[j, j]) + 1.0
    qr_ref, tau_ref, twy_ref = oracle.hqr(a)
    assert np.sum(tau_ref == 0.0) >= 3
    A = cm_cuda(a)
    tau = torch.zeros(p, dtype=torch.float64, device="cuda")
    twy = cm_empty(p, p)
    rutv.hqr(A, tau, twy)
    assert np.max(np.abs(tau.cpu().numpy() - tau_ref)) < 1e-12
    assert np.max(np.abs(to_np(twy) - twy_ref)) < 1e-10
    # and a panel with every tau != 0 through the inverse form, against the recurrence
    b = oracle.gaussian_matrix(500, 100, 18)
    _, tau_b, twy_b = oracle.hqr(b)
    B = cm_cuda(b)
    tb = torch.zeros(100, dtype=torch.float64, device="cuda")
    tw = cm_empty(100, 100)
    rutv.hqr(B, tb, tw)
    assert np.max(np.abs(to_np(tw) - twy_b)) < 1e-10 * max(1.0, np.max(np.abs(twy_b)))
