"""End-to-end parity of the B200 randUTV against the CPU oracle (C ABI calls).

Small sizes: entrywise parity after sign alignment, with the reference's own
Gaussian stream passed explicitly (bit-identical inputs).  Invariants follow
test_randutv_blocked.cpp:40-78 and acceptance.cpp:91-165.
"""
import numpy as np
import pytest

import oracle
import paper_2104_05782_b200 as rutv
from tests._util import check_structure, compare_to_oracle, orth_defect, residual

pytestmark = pytest.mark.gpu


def _run(a, b, q, seed, explicit_g=True, **kw):
    m, n = a.shape
    g = oracle.normal_stream(seed, 0, oracle.stream_length(m, n, b)) if explicit_g else None
    return rutv.factorize(a, b=b, q=q, seed=seed, g=g, **kw)


@pytest.mark.parametrize("n,b,q", [(24, 8, 1), (25, 8, 1), (16, 4, 0), (6, 8, 1), (64, 16, 0),
                                   (64, 16, 2), (100, 32, 1), (127, 16, 2), (256, 64, 1),
                                   (300, 128, 0), (520, 128, 2)])
def test_factorize_matches_oracle_small(n, b, q):
    a = oracle.gaussian_matrix(n, n, 300 + 31 * n + n)
    got = _run(a, b, q, 7)
    ref = oracle.randutv(a, b=b, q=q, seed=7)
    t, u, v = got
    check_structure(t, b)
    assert residual(a, t, u, v) < 1e-13
    assert orth_defect(u) < 1e-12 and orth_defect(v) < 1e-12
    compare_to_oracle(a, got, ref)


def test_factorize_device_rng_close_to_oracle():
    n, b, q = 200, 32, 1
    a = oracle.gaussian_matrix(n, n, 5)
    t, u, v = _run(a, b, q, 3, explicit_g=False)
    ref = oracle.randutv(a, b=b, q=q, seed=3)
    check_structure(t, b)
    compare_to_oracle(a, (t, u, v), ref, t_tol=1e-10, uv_tol=1e-8, diag_rel=1e-9)


def test_factorize_no_uv_same_t():
    a = oracle.gaussian_matrix(96, 96, 330)
    g = oracle.normal_stream(11, 0, oracle.stream_length(96, 96, 16))
    t1, u1, v1 = rutv.factorize(a, b=16, q=1, seed=11, g=g, build_uv=False)
    t2, _, _ = rutv.factorize(a, b=16, q=1, seed=11, g=g)
    assert u1 is None and v1 is None
    assert np.array_equal(t1, t2)


def test_factorize_deterministic():
    a = oracle.gaussian_matrix(300, 300, 320)
    r1 = rutv.factorize(a, b=64, q=1, seed=11)
    r2 = rutv.factorize(a, b=64, q=1, seed=11)
    for x, y in zip(r1, r2):
        assert np.array_equal(x, y)
    r3 = rutv.factorize(a, b=64, q=1, seed=12)
    assert not np.array_equal(r1[0], r3[0])


def test_diag_4321_recovery():
    # test_randutv_blocked.cpp:111-137
    a = np.diag([4.0, 3.0, 2.0, 1.0])
    t, u, v = _run(a, 2, 2, 5)
    check_structure(t, 2)
    st = np.linalg.svd(t, compute_uv=False)
    assert np.max(np.abs(st - [4, 3, 2, 1])) < 1e-10
    ref = oracle.randutv(a, b=2, q=2, seed=5)
    compare_to_oracle(a, (t, u, v), ref)


def test_degenerate_shapes():
    t, u, v = rutv.factorize(np.zeros((0, 0)), b=4)
    assert t.shape == (0, 0)
    t, u, v = rutv.factorize(np.array([[-3.5]]), b=4)
    assert abs(t[0, 0] - 3.5) < 1e-15 and abs(abs(u[0, 0]) - 1.0) < 1e-15


def test_config_errors():
    a = oracle.gaussian_matrix(8, 8, 360)
    # b <= 0 selects the default 128 exactly like the reference binding
    # (bindings.cpp:55: cfg.b = b > 0 ? b : 128); q < 0 is a ConfigError -> ValueError
    t, _, _ = rutv.factorize(a, b=-1)
    t2, _, _ = rutv.factorize(a, b=128)
    assert np.array_equal(t, t2)
    with pytest.raises(ValueError):
        rutv.factorize(a, b=4, q=-1)


@pytest.mark.parametrize("kind", ["gaussian", "geometric"])
def test_config1_shape_invariants(kind):
    """n = 1000 slice of configs 1 / 2 (full configs run in test_gpu_configs.py)."""
    n, b, q = 1000, 128, 2
    a = (oracle.gaussian_matrix(n, n, 1) if kind == "gaussian"
         else oracle.geometric_matrix(n, n, 10 ** (-12 / (n - 1)), 1))
    t, u, v = _run(a, b, q, 2)
    check_structure(t, b)
    assert residual(a, t, u, v) < 1e-12
    assert orth_defect(u) < 1e-11 and orth_defect(v) < 1e-11
    sa = np.linalg.svd(a, compute_uv=False)
    st = np.linalg.svd(t, compute_uv=False)
    assert np.max(np.abs(sa - st)) < 1e-11 * sa[0]


def test_overlap_is_bit_identical():
    """Two-stream schedule == single-stream schedule, bit for bit."""
    import os
    a = oracle.gaussian_matrix(700, 700, 77)
    r1 = rutv.factorize(a, b=64, q=1, seed=3)
    os.environ["RUTV_OVERLAP"] = "0"
    try:
        r2 = rutv.factorize(a, b=64, q=1, seed=3)
    finally:
        os.environ.pop("RUTV_OVERLAP")
    for x, y in zip(r1, r2):
        assert np.array_equal(x, y)


def test_cpp_dropin_shim_runs(tmp_path):
    import subprocess
    from tests.test_capi import _build_shim
    exe = _build_shim(str(tmp_path / "shim"))
    out = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "config_error=1" in out.stdout
