"""The micro-panel fast path of the cluster panel-QR kernel (qr_reg.cu "CQ": Cholesky-QR2 +
Householder reconstruction of full 16-column micro-panels) against the reference's
hqr_inplace (householder.cpp:48-67) through the oracle, in every mode of the path
(RUTV_QR_CQ is read once per process, hence subprocesses):
  1  default: CQ micro-panels, column loop only where a micro-panel is unsafe / ragged;
  0  column loop only (the round-1 kernel);
  2  every odd micro-panel takes the pass-2 recovery (X restored as X1 R1, then the column loop);
  3  every odd micro-panel takes the pass-1 fallback (registers untouched).
RUTV_CHOLQR_MIN_ROWS=0 keeps tall panels on this kernel, which exercises two rows per thread."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

SCRIPT = r'''
import sys, json
sys.path.insert(0, ".")
import numpy as np, torch
import oracle, paper_2104_05782_b200 as rutv
from tests._util import cm_cuda, cm_empty, to_np
out = []
for s, w, kind in ((2000, 128, "gauss"), (4000, 128, "gauss"), (700, 100, "gauss"), (130, 48, "gauss"), (64, 64, "gauss"),
                   (9000, 64, "gauss"), (300, 64, "graded"), (96, 32, "tri"), (500, 48, "tiny"), (500, 48, "huge")):
    if kind == "gauss":
        y = oracle.gaussian_matrix(s, w, 7)
    elif kind == "graded":  # columns scaled over 12 decades: the Gram matrix of a micro-panel is ill-conditioned
        y = oracle.gaussian_matrix(s, w, 8) * np.logspace(0, -12, w)[None, :]
    elif kind == "tiny":    # X'X ~ 1e-282: outside the pivot range the Gram path accepts -> column loop
        y = oracle.gaussian_matrix(s, w, 9) * 1e-142  # (the reference's own sum of squares is still normal)
    elif kind == "huge":    # X'X ~ 1e284
        y = oracle.gaussian_matrix(s, w, 9) * 1e141
    else:                   # already triangular: tau = 0 reflectors (LU pivot 0 -> column loop)
        y = np.triu(np.ones((s, w)))
    p = min(s, w)
    a = cm_cuda(y); tau = torch.zeros(p, dtype=torch.float64, device="cuda"); twy = cm_empty(p, p)
    rutv.hqr(a, tau, twy)
    qr_ref, tau_ref, twy_ref = oracle.hqr(y)
    g = to_np(a)
    cs = np.maximum(np.max(np.abs(qr_ref[:p]), axis=0), 1e-300)  # column scale of R (graded case)
    out.append({"s": s, "w": w, "kind": kind,
                "r": float(np.max(np.abs(np.triu(g[:p]) - np.triu(qr_ref[:p])) / cs[None, :])),
                "v": float(np.max(np.abs(np.tril(g, -1) - np.tril(qr_ref, -1)))),
                "tau": float(np.max(np.abs(tau.cpu().numpy() - tau_ref))),
                "twy": float(np.max(np.abs(to_np(twy) - twy_ref)))})
print(json.dumps(out))
'''


@pytest.mark.parametrize("mode", ["1", "0", "2", "3"])
def test_cq_micro_panels_match_oracle(mode):
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, RUTV_QR_CQ=mode, RUTV_CHOLQR_MIN_ROWS="0")
    res = subprocess.run([sys.executable, "-c", SCRIPT], cwd=root, env=env, capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stderr[-2000:]
    for r in json.loads(res.stdout.strip().splitlines()[-1]):
        if r["kind"] == "tri":
            assert r["r"] == 0.0 and r["v"] == 0.0 and r["tau"] == 0.0, r  # returned bit-equal, tau = 0
        else:
            assert r["r"] < 1e-12 and r["v"] < 1e-11 and r["tau"] < 1e-12 and r["twy"] < 1e-10, r  # NaN fails too
