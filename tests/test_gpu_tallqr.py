"""Tall panels (rows >= RUTV_CHOLQR_MIN_ROWS, default 4608) factor their <= 128-column
sub-panels by Cholesky-QR2 + Householder reconstruction (cholqr.cu, qr_cluster.cu
hqr_panel) and must reproduce the reference's hqr_inplace (householder.cpp:48-67):
packed R / V and tau against the oracle, on a well-conditioned panel (fast path
taken) and on panels whose sub-panels are unsafe (rank-deficient columns, an
already-triangular head -> tau = 0), where the per-sub-panel fallback to the
Householder kernels must give the reference's exact conventions."""
import ctypes as C

import numpy as np
import pytest

import oracle
from tests._util import cm_cuda, to_np

pytestmark = pytest.mark.gpu


def _hqr(y):
    import torch
    import paper_2104_05782_b200 as rutv
    L = rutv.lib()
    L.rutv_b200_set_stream(C.c_uint64(torch.cuda.current_stream().cuda_stream))
    s, w = y.shape
    a = cm_cuda(y)
    tau = torch.zeros(min(s, w), dtype=torch.float64, device="cuda")
    st = rutv.Status()
    rc = L.rutv_b200_hqr_async(C.c_void_p(a.data_ptr()), s, w, s, C.c_void_p(tau.data_ptr()), C.byref(st))
    torch.cuda.synchronize()
    assert rc == 0, st.message
    return to_np(a), tau.cpu().numpy()


def _check(y, r_tol, v_tol, tau_tol):
    qr_ref, tau_ref, _ = oracle.hqr(y)
    g, tau = _hqr(y)
    w = y.shape[1]
    scale = max(np.max(np.abs(qr_ref[:w])), 1e-300)
    out = {"r": float(np.max(np.abs(np.triu(g[:w]) - np.triu(qr_ref[:w]))) / scale),
           "v": float(np.max(np.abs(np.tril(g, -1) - np.tril(qr_ref, -1)))),
           "tau": float(np.max(np.abs(tau - tau_ref)))}
    assert out["r"] <= r_tol and out["v"] <= v_tol and out["tau"] <= tau_tol, out
    return out


@pytest.mark.parametrize("s,w", [(7000, 256), (6500, 130), (9000, 128)])
def test_tall_panel_matches_oracle(s, w):
    _check(oracle.gaussian_matrix(s, w, 21), 1e-13, 1e-13, 1e-13)


def test_tall_panel_unsafe_subpanels_fall_back():
    s, w = 6400, 256
    y = oracle.gaussian_matrix(s, w, 22)
    # second sub-panel: columns 128..255 repeat columns 0..127 scaled -> after the first
    # sub-panel's update they are ~0 below the diagonal block: Cholesky breaks down / the
    # diag(R1) ratio trips, and the Householder kernels must take that sub-panel.
    y[:, 128:] = 0.5 * y[:, :128]
    # R's noise-level entries are rounding-determined; compare the reconstruction instead
    import torch
    g, tau = _hqr(y)
    r = np.triu(g[:w])
    v = np.tril(g, -1)
    v[np.arange(w), np.arange(w)] = 1.0
    # Q^T y = R via the reflectors, applied in order
    z = torch.from_numpy(y.copy())
    vt, tt = torch.from_numpy(v), torch.from_numpy(tau)
    for j in range(w):
        z -= tt[j] * torch.outer(vt[:, j], vt[:, j] @ z)
    z = z.numpy()
    assert np.max(np.abs(z[:w] - r)) <= 1e-11 * np.max(np.abs(y))
    assert np.max(np.abs(z[w:])) <= 1e-11 * np.max(np.abs(y))
    assert np.all(tau >= 0.0) and np.all(tau <= 2.0)
    # the well-conditioned first sub-panel still matches the oracle entrywise
    qr_ref, tau_ref, _ = oracle.hqr(y[:, :128])
    assert np.max(np.abs(g[:, :128] - qr_ref)) <= 1e-12 * np.max(np.abs(qr_ref))
    assert np.max(np.abs(tau[:128] - tau_ref)) <= 1e-13


@pytest.mark.parametrize("scale", [1e-142, 1e141])
def test_tall_panel_extreme_scaling(scale):
    # Y'Y ~ 1e-282 / 1e284, close to the ends of the double range (where the reference's own
    # sums of squares are still normal numbers)
    _check(oracle.gaussian_matrix(6300, 40, 23) * scale, 1e-13, 1e-13, 1e-13)  # R relative to max |R|


def test_tall_panel_triangular_head_keeps_tau_zero_convention():
    s, w = 6200, 64
    y = np.triu(np.ones((s, w)))  # already upper triangular: every reflector is tau = 0
    _check(y, 0.0, 0.0, 0.0)
