"""The opt-in Cholesky-QR2 + Householder-reconstruction panel QR (cholqr.cu)
against the oracle's Householder QR (householder.cpp:48-67), in a subprocess
with RUTV_CHOLQR=1 (the switch is read once per process)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

SCRIPT = r'''
import ctypes as C, sys, json
sys.path.insert(0, ".")
import numpy as np, torch
import oracle, paper_2104_05782_b200 as rutv
from tests._util import cm_cuda, to_np
L = rutv.lib()
L.rutv_b200_set_stream(C.c_uint64(torch.cuda.current_stream().cuda_stream))
out = []
for s, p, kind in ((2000, 128, "gauss"), (700, 100, "gauss"), (300, 37, "gauss"), (64, 16, "tri")):
    Y = oracle.gaussian_matrix(s, p, 3) if kind == "gauss" else np.triu(np.ones((s, p)))
    A = cm_cuda(Y); tau = torch.zeros(p, dtype=torch.float64, device="cuda")
    st = rutv.Status()
    rc = L.rutv_b200_hqr_async(C.c_void_p(A.data_ptr()), s, p, s, C.c_void_p(tau.data_ptr()), C.byref(st))
    torch.cuda.synchronize()
    qr_ref, tau_ref, _ = oracle.hqr(Y)
    g = to_np(A)
    out.append({"s": s, "p": p, "rc": rc,
                "r": float(np.max(np.abs(np.triu(g[:p]) - np.triu(qr_ref[:p]))) / max(1e-300, np.max(np.abs(qr_ref)))),
                "v": float(np.max(np.abs(np.tril(g, -1) - np.tril(qr_ref, -1)))),
                "tau": float(np.max(np.abs(tau.cpu().numpy() - tau_ref)))})
print(json.dumps(out))
'''


def test_cholqr_fast_path_matches_householder():
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, RUTV_CHOLQR="1")
    res = subprocess.run([sys.executable, "-c", SCRIPT], cwd=root, env=env, capture_output=True, text=True,
                         timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    import json
    rows = json.loads(res.stdout.strip().splitlines()[-1])
    for r in rows:
        # the already-triangular panel has tau = 0 reflectors -> the guarded
        # fallback (Householder kernel) runs; either way the result must match
        assert r["rc"] == 0 and r["r"] < 1e-13 and r["v"] < 1e-12 and r["tau"] < 1e-12, r


DEFERRED = r'''
import sys, json
sys.path.insert(0, ".")
import numpy as np
import oracle, paper_2104_05782_b200 as rutv
out = []
def run(a, b, q, seed):
    n = a.shape[0]
    g = oracle.normal_stream(seed, 0, oracle.stream_length(n, n, b))
    t, u, v = rutv.factorize(a, b=b, q=q, seed=seed, g=g)
    tr, ur, vr = oracle.randutv(a, b=b, q=q, seed=seed)
    d = np.sign(np.einsum("ij,ij->j", u, ur)); d[d == 0] = 1
    nf = np.linalg.norm(a)
    return {"t": float(np.max(np.abs(t - d[:, None] * tr * d[None, :])) / nf),
            "diag": float(np.max(np.abs(np.abs(np.diag(t)) - np.abs(np.diag(tr))) / np.maximum(np.abs(np.diag(tr)), 1e-300))),
            "resid": float(np.linalg.norm(a - u @ t @ v.T) / nf),
            "orth": float(max(np.max(np.abs(u.T @ u - np.eye(n))), np.max(np.abs(v.T @ v - np.eye(n)))))}
out.append(run(oracle.gaussian_matrix(520, 520, 11), 64, 1, 5))
# rank 200: trailing panels are exactly rank deficient -> unsafe Cholesky-QR2 -> Householder re-run
x = oracle.gaussian_matrix(520, 200, 12); y = oracle.gaussian_matrix(200, 520, 13)
out.append(run(x @ y, 64, 1, 5))
print(json.dumps(out))
'''


def test_cholqr_deferred_driver_and_rerun():
    """RUTV_CHOLQR=2: the factorization driver's deferred Cholesky-QR2 panels
    (no host synchronisation per panel) match the oracle; a rank-deficient
    input trips the device safety flag and the driver re-runs with Householder."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, RUTV_CHOLQR="2", RUTV_DEBUG="1")
    res = subprocess.run([sys.executable, "-c", DEFERRED], cwd=root, env=env, capture_output=True, text=True,
                         timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    import json
    full, lowrank = json.loads(res.stdout.strip().splitlines()[-1])
    assert full["t"] < 1e-11 and full["diag"] < 1e-10 and full["resid"] < 1e-13 and full["orth"] < 1e-12, full
    assert lowrank["resid"] < 1e-13 and lowrank["orth"] < 1e-12, lowrank
    assert "re-running with Householder" in res.stderr
