"""Shared helpers for the parity tests (test infrastructure)."""
from __future__ import annotations

import numpy as np


def cm_cuda(x: np.ndarray, device: int = 0):
    """numpy (m x n) -> column-major fp64 CUDA tensor view (stride (1, m))."""
    import torch
    x = np.asarray(x, dtype=np.float64)
    m, n = x.shape
    t = torch.empty((n, m), dtype=torch.float64, device=f"cuda:{device}")
    t.copy_(torch.from_numpy(np.ascontiguousarray(x.T)))
    return t.T


def cm_empty(m: int, n: int, device: int = 0, fill: float = 0.0):
    import torch
    return torch.full((n, m), fill, dtype=torch.float64, device=f"cuda:{device}").T


def to_np(t) -> np.ndarray:
    return np.asfortranarray(t.detach().cpu().numpy())


def sign_align(u_gpu, u_ref):
    """D = diag(sign <u_gpu(:,k), u_ref(:,k)>)."""
    d = np.sign(np.einsum("ij,ij->j", u_gpu, u_ref))
    d[d == 0] = 1.0
    return d


def orth_defect(q: np.ndarray) -> float:
    return float(np.linalg.norm(q.T @ q - np.eye(q.shape[1])))


def residual(a, t, u, v) -> float:
    return float(np.linalg.norm(a - u @ t @ v.T) / max(np.linalg.norm(a), 1e-300))


def check_structure(t: np.ndarray, b: int) -> None:
    """Invariants of test_randutv_blocked.cpp:52-66: strictly-lower T exactly 0,
    each b x b diagonal window exactly diagonal, non-increasing, >= 0."""
    m, n = t.shape
    assert np.all(np.tril(t, -1) == 0.0), "strictly-lower T must be exact zeros"
    p = min(m, n)
    for r0 in range(0, p, b):
        w = min(b, p - r0)
        blk = t[r0:r0 + w, r0:r0 + w]
        off = blk - np.diag(np.diag(blk))
        assert np.all(off == 0.0), f"diagonal window at {r0} not exactly diagonal"
        d = np.diag(blk)
        assert np.all(d[:-1] >= d[1:]), f"window at {r0} not sorted"
        assert d[-1] >= 0.0


def compare_to_oracle(a, got, ref, *, t_tol=1e-11, uv_tol=1e-9, diag_rel=1e-10):
    """Sign-aligned entrywise parity of (T, U, V) against the oracle."""
    tg, ug, vg = got
    tr, ur, vr = ref
    nf = np.linalg.norm(a)
    d = sign_align(ug, ur) if ug is not None else np.ones(tg.shape[1])
    tr_al = d[:, None] * tr * d[None, :] if tg.shape[0] == tg.shape[1] else tr
    dt = float(np.max(np.abs(tg - tr_al))) / nf
    out = {"t_maxabs_rel": dt}
    dg, dr = np.diag(tg), np.diag(tr)
    out["diag_rel"] = float(np.max(np.abs(dg - dr) / np.maximum(np.abs(dr), 1e-300)))
    if ug is not None:
        out["u_maxabs"] = float(np.max(np.abs(ug - ur * d[None, :])))
        out["v_maxabs"] = float(np.max(np.abs(vg - vr * d[None, :])))
    assert dt <= t_tol, out
    assert out["diag_rel"] <= diag_rel, out
    if ug is not None:
        assert out["u_maxabs"] <= uv_tol and out["v_maxabs"] <= uv_tol, out
    return out


def cluster_align(ug, ur, d_ref, b, rel=1e-8):
    """Alignment D (n x n, block diagonal) with ug ~= ur @ D for comparing two
    randUTV runs.

    Each step's Jacobi SVD fixes (u_k, v_k) pairs only up to sign -- and, inside a
    cluster of (near-)equal singular values of one b x b window (config 4's
    sigma = 1 block), only up to an orthogonal rotation, because the order after
    the stable sort of jacobi_svd.cpp:111-122 and the basis inside the cluster
    are rounding-determined.  Within every window, consecutive indices whose
    reference diagonal agrees to `rel` form a cluster; a singleton gets the sign
    of <ug_k, ur_k>, a cluster the orthogonal Procrustes factor polar(ur_c' ug_c).
    Then U_gpu ~ U_ref D, V_gpu ~ V_ref D and T_gpu ~ D' T_ref D."""
    n = ug.shape[1]
    D = np.zeros((n, n))
    for r0 in range(0, n, b):
        w = min(b, n - r0)
        i = r0
        while i < r0 + w:
            j = i + 1
            while j < r0 + w and abs(d_ref[j] - d_ref[i]) <= rel * max(abs(d_ref[i]), 1e-300):
                j += 1
            if j - i == 1:
                s = np.sign(ug[:, i] @ ur[:, i])
                D[i, i] = s if s != 0 else 1.0
            else:
                m = ur[:, i:j].T @ ug[:, i:j]
                w_, _, zt = np.linalg.svd(m)
                D[i:j, i:j] = w_ @ zt
            i = j
    return D
