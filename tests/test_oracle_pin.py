"""Pins the CPU oracle (oracle/rutv_oracle.c) -- CPU only.

1. Against the committed golden fixtures made by the unmodified reference
   (tests/golden/make_golden.py): bit-exact, runs anywhere.
2. Against the reference compiled here (oracle/_ref), when /root/reference is
   present: bit-exact on shapes from test_randutv_blocked.cpp:83-88 and
   acceptance.cpp:96-99, including ragged, trapezoidal and qr_prepass cases.
3. The reference's own known-answer checks (test_householder.cpp:114-130,
   test_block_svd.cpp:131-141, test_matrix.cpp:266-278).
"""
import glob
import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _load(name):
    return np.load(os.path.join(GOLD, name))


def test_golden_rng_bit_exact():
    g = _load("rng.npz")
    assert np.array_equal(oracle.normal_stream(42, 0, 64), g["seed42_pos0"])
    assert np.array_equal(oracle.normal_stream(7, 10**9, 64), g["seed7_pos1e9"])
    assert np.array_equal(oracle.normal_stream(0, 0, 64), g["seed0_pos0"])


def test_golden_gemm_bit_exact():
    g = _load("gemm.npz")
    for ta in (0, 1):
        for tb in (0, 1):
            a = g["a"].T.copy() if ta else g["a"]
            b = g["b"].T.copy() if tb else g["b"]
            got = oracle.gemm(-0.75, ta, a, tb, b, 0.5, g["c0"])
            assert np.array_equal(got, g[f"c_{ta}{tb}"])


def test_golden_hqr_bit_exact():
    g = _load("hqr.npz")
    for name in ["g9x4", "g40x12", "tri4", "neghead3", "zero_col5x3"]:
        qr, tau, twy = oracle.hqr(g[name + "_a"])
        assert np.array_equal(qr, g[name + "_qr"]), name
        assert np.array_equal(tau, g[name + "_tau"]), name
        assert np.array_equal(twy, g[name + "_twy"]), name


def test_golden_svd_bit_exact():
    g = _load("svd.npz")
    for name in ["k2x2", "g6", "g16", "shuffled_diag4", "rank1_5"]:
        u, s, v = oracle.svd_block(g[name + "_a"])
        assert np.array_equal(u, g[name + "_u"]), name
        assert np.array_equal(s, g[name + "_s"]), name
        assert np.array_equal(v, g[name + "_v"]), name


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(GOLD, "randutv_*.npz"))))
def test_golden_randutv_bit_exact(path):
    g = np.load(path)
    m, n, b, q, seed = (int(x) for x in g["meta"])
    t, u, v = oracle.randutv(g["a"], b=b, q=q, seed=seed)
    assert np.array_equal(t, g["t"])
    assert np.array_equal(u, g["u"])
    assert np.array_equal(v, g["v"])


def test_known_answers():
    # 2x2 Jacobi: sigma = sqrt(45), sqrt(5)  (test_block_svd.cpp:131-141)
    _, s, _ = oracle.svd_block(np.array([[3.0, 0.0], [4.0, 5.0]]))
    assert abs(s[0] - np.sqrt(45)) < 1e-14 * 7 and abs(s[1] - np.sqrt(5)) < 1e-14 * 3
    # triangular input: tau = 0 and bit-equal output (test_householder.cpp:114-121)
    a = np.triu(np.add.outer(np.arange(4), np.arange(4)) + 1.0)
    qr, tau, _ = oracle.hqr(a)
    assert np.all(tau == 0.0) and np.array_equal(qr, a)
    # negative head without tail: tau = 2, R = +2 (test_householder.cpp:123-130)
    qr, tau, _ = oracle.hqr(np.diag([-2.0, 1.0, 1.0]))
    assert qr[0, 0] == 2.0 and tau[0] == 2.0
    # tau * v'v == 2 (test_householder.cpp:104-112)
    qr, tau, _ = oracle.hqr(oracle.gaussian_matrix(7, 4, 11))
    for j in range(4):
        vtv = 1.0 + np.sum(qr[j + 1:, j] ** 2)
        assert abs(tau[j] * vtv - 2.0) < 1e-12
    # column-major stream consumption (test_matrix.cpp:266-278)
    a = oracle.gaussian_matrix(3, 2, 5)
    st = oracle.normal_stream(5, 0, 6)
    assert a[0, 0] == st[0] and a[2, 0] == st[2] and a[0, 1] == st[3]


def test_config_error_codes():
    a = oracle.gaussian_matrix(8, 8, 360)
    with pytest.raises(oracle.OracleError) as e:
        oracle.randutv(a, b=0)
    assert e.value.code == 1
    with pytest.raises(oracle.OracleError) as e:
        oracle.randutv(a, b=4, q=-1)
    assert e.value.code == 1
    with pytest.raises(oracle.OracleError) as e:
        oracle.svd_block(oracle.gaussian_matrix(6, 6, 230), max_sweeps=0)
    assert e.value.code == 4 and e.value.residual > 0


def test_flop_model_matches_survey():
    want = [7.4785e10, 7.3549e11, 9.9453e12, 2.9398e14, 1.3664e15]
    got = [oracle.flops(n, b, q) for n, b, q in
           [(2000, 128, 0), (4000, 128, 2), (10000, 256, 1), (30000, 256, 2), (50000, 512, 2)]]
    for g, w in zip(got, want):
        assert abs(g - w) / w < 1e-4


ref_only = pytest.mark.skipif(not oracle.available("ref"), reason="oracle/_ref not built")


@ref_only
@pytest.mark.parametrize("m,n,b,q", [(24, 24, 8, 1), (30, 20, 8, 0), (20, 30, 8, 2), (25, 25, 8, 1),
                                     (13, 7, 5, 1), (6, 6, 8, 1), (16, 16, 4, 0), (64, 64, 8, 0),
                                     (96, 48, 16, 1), (48, 96, 16, 2), (100, 64, 8, 2),
                                     (200, 200, 64, 1)])
def test_port_equals_reference(m, n, b, q):
    a = oracle.gaussian_matrix(m, n, 300 + m * 31 + n, impl="ref")
    for qp in (False, True):
        r1 = oracle.randutv(a, b=b, q=q, seed=7, qr_prepass=qp)
        r2 = oracle.randutv(a, b=b, q=q, seed=7, qr_prepass=qp, impl="ref")
        for x, y in zip(r1, r2):
            assert np.array_equal(x, y)


@ref_only
def test_step_limited_reference_replica_is_exact():
    """ref_randutv_steps (public step API) == randutv() and == the port, per k."""
    a = oracle.gaussian_matrix(120, 120, 9, impl="ref")
    full = oracle.randutv(a, b=32, q=1, seed=4, impl="ref")
    rep = oracle.randutv(a, b=32, q=1, seed=4, impl="ref", max_steps=100)
    for x, y in zip(full, rep):
        assert np.array_equal(x, y)
    for k in (1, 2, 3):
        r1 = oracle.randutv(a, b=32, q=1, seed=4, impl="ref", max_steps=k)
        r2 = oracle.randutv(a, b=32, q=1, seed=4, max_steps=k)
        for x, y in zip(r1, r2):
            assert np.array_equal(x, y)


@ref_only
def test_generators_equal_reference():
    assert np.array_equal(oracle.gaussian_matrix(50, 40, 3), oracle.gaussian_matrix(50, 40, 3, impl="ref"))
    assert np.array_equal(oracle.geometric_matrix(60, 60, 0.9, 3),
                          oracle.geometric_matrix(60, 60, 0.9, 3, impl="ref"))
    assert np.array_equal(oracle.normal_stream(5, 12345, 500), oracle.normal_stream(5, 12345, 500, impl="ref"))


@pytest.mark.skipif(not oracle.available("ref"), reason="reference library not built")
def test_reference_ab_driver_for_cpu_baseline():
    # bench.py's CPU baseline also times the reference's multi-threaded algorithm-by-blocks
    # driver (randutv_ab.hpp:46): same contract as randutv(), bitwise identical for any
    # worker count, b | n required.
    a = oracle.geometric_matrix(64, 64, 0.9, 3, impl="ref")
    t1, u1, v1 = oracle.ref_randutv_ab(a, b=16, q=1, seed=2, workers=1)
    t4, u4, v4 = oracle.ref_randutv_ab(a, b=16, q=1, seed=2, workers=4)
    assert np.array_equal(t1, t4) and np.array_equal(u1, u4) and np.array_equal(v1, v4)
    assert np.linalg.norm(a - u1 @ t1 @ v1.T) / np.linalg.norm(a) < 1e-13
    assert np.all(np.tril(t1, -1) == 0.0)
    with pytest.raises(oracle.OracleError):
        oracle.ref_randutv_ab(oracle.gaussian_matrix(60, 60, 1), b=16, q=1, seed=2, workers=2)
