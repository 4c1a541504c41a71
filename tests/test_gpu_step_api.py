"""The public step API (randutv_blocked.hpp:41-72) on the B200 through the C ABI.

The reference's own replay (oracle/ref_shim.cpp ref_randutv_steps, bit-identical to
randutv()) drives the loop of randutv_blocked.cpp:114-155 through build_v_alpha /
apply_q_right / build_u_alpha / apply_qt_left / beta_stage.  The same replay with
OUR build_v_alpha / build_u_alpha / beta_stage (the applies in the oracle, the
reference's G passed explicitly) must reproduce the oracle's first-k-step state.
"""
import numpy as np
import pytest

import oracle
import paper_2104_05782_b200 as rutv
from tests._util import compare_to_oracle

pytestmark = pytest.mark.gpu


def _replay(a, b, q, seed, steps):
    m, n = a.shape
    t = np.asfortranarray(a.copy())
    u, v = np.eye(m, order="F"), np.eye(n, order="F")
    pos = 0
    for i in range(steps):
        r0 = i * b
        rr, cr = m - r0, n - r0
        if rr <= 0 or cr <= 0 or cr <= b:
            break
        t22 = np.asfortranarray(t[r0:, r0:])
        g = oracle.normal_stream(seed, pos, rr * b)
        qr, tau, twy = rutv.build_v_alpha(t22, b, q, seed, pos, g=g)
        pos += rr * b
        t[r0:, r0:] = oracle.apply_q_right(qr, twy, t[r0:, r0:])
        if r0 > 0:
            t[:r0, r0:] = oracle.apply_q_right(qr, twy, t[:r0, r0:])
        v[:, r0:] = oracle.apply_q_right(qr, twy, v[:, r0:])
        panel = np.asfortranarray(t[r0:, r0:r0 + b])
        qru, tauu, twyu = rutv.build_u_alpha(panel)
        t[r0:, r0:r0 + b] = panel
        t[r0:, r0 + b:] = oracle.apply_qt_left(qru, twyu, t[r0:, r0 + b:])
        u[:, r0:] = oracle.apply_q_right(qru, twyu, u[:, r0:])
        t22 = np.asfortranarray(t[r0:, r0:])
        bu, bv = rutv.beta_stage(t22, b)
        t[r0:, r0:] = t22
        if r0 > 0:
            t[:r0, r0:r0 + b] = t[:r0, r0:r0 + b] @ bv
        u[:, r0:r0 + bu.shape[0]] = u[:, r0:r0 + bu.shape[0]] @ bu
        v[:, r0:r0 + b] = v[:, r0:r0 + b] @ bv
    return t, u, v


@pytest.mark.parametrize("n,b,q,steps", [(64, 16, 1, 2), (100, 32, 2, 3), (130, 48, 0, 2), (300, 64, 1, 1)])
def test_step_api_replay_matches_oracle(n, b, q, steps):
    a = oracle.gaussian_matrix(n, n, 1000 + n)
    got = _replay(a, b, q, 9, steps)
    ref = oracle.randutv(a, b=b, q=q, seed=9, max_steps=steps)
    # the unfinished trailing block's diagonal is raw (not yet SVD'd) and may be tiny: the
    # pure-relative diag test applies to the finished windows.  The n = 100, q = 2 case ends on a
    # 36 x 36 trailing block whose sketch (T22'T22)^2 T22'G is ill-conditioned: ANY backward-stable
    # panel QR moves Q by eps * cond(Y) there (the column-by-column Householder kernel differs from
    # the oracle by 4.7e-13 / 7.8e-11 in T / V, the Cholesky-QR2 micro-panels by 1.0e-12 / 1.1e-10;
    # every well-conditioned case agrees to 1e-15 / 1e-13 with either, tools/chk_stepapi.py)
    loose = (n, q) == (100, 2)
    compare_to_oracle(a, got, ref, t_tol=5e-12 if loose else 1e-12, uv_tol=5e-10 if loose else 1e-10, diag_rel=1e-6)
    k = min(steps * b, n)
    dg, dr = np.diag(got[0])[:k], np.diag(ref[0])[:k]
    assert np.max(np.abs(dg - dr) / np.abs(dr)) <= 1e-10


def test_build_v_alpha_device_rng_and_position():
    n, b, q = 80, 16, 1
    a = oracle.gaussian_matrix(n, n, 3)
    g = oracle.normal_stream(5, 1000, n * b)
    qr1, tau1, twy1 = rutv.build_v_alpha(a, b, q, 5, 1000, g=g)
    qr2, tau2, twy2 = rutv.build_v_alpha(a, b, q, 5, 1000)  # device-drawn deviates from the same position
    assert np.max(np.abs(qr1 - qr2)) < 1e-10 and np.max(np.abs(tau1 - tau2)) < 1e-12
    assert tau1.shape == (b,) and twy1.shape == (b, b)
    assert np.all(np.tril(twy1, -1) == 0) and np.allclose(np.diag(twy1), tau1)
    # host RngState mirror (the drop-in header's RngState::normal_at) is the reference stream
    assert all(rutv.normal_at(5, d) == x for d, x in zip(range(1000, 1010), g[:10]))


def test_beta_stage_trapezoid_and_errors():
    rows, cols, bw = 5, 12, 8  # rt = rows < bw: the trapezoidal case (randutv_blocked.cpp:71)
    t22 = np.asfortranarray(np.triu(oracle.gaussian_matrix(rows, cols, 4)))
    before = t22.copy()
    u, v = rutv.beta_stage(t22, bw)
    assert u.shape == (5, 5) and v.shape == (8, 8)
    expected = np.zeros((rows, bw))
    expected[np.arange(rows), np.arange(rows)] = np.diag(t22)[:rows]
    assert np.array_equal(t22[:, :bw], expected)  # write_rect_diag: everything else exactly 0
    s = np.diag(t22)[:rows]
    assert np.all(s[:-1] >= s[1:]) and s[-1] >= 0
    r = np.triu(before[:, :bw])
    assert np.allclose(u @ t22[:, :bw] @ v.T, r, atol=1e-13)
    assert np.allclose(t22[:, bw:], u.T @ before[:, bw:], atol=1e-13)
    with pytest.raises(ValueError):
        rutv.beta_stage(np.asfortranarray(before.copy()), cols + 1)
    with pytest.raises(ValueError):
        rutv.build_v_alpha(before, 0, 1, 0, 0)
