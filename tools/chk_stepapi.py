"""Deviation of the step-API replay from the oracle (tests/test_gpu_step_api.py cases), for A/B
runs of the panel-QR paths (RUTV_QR_CQ=0/1)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
from tests.test_gpu_step_api import _replay
from tests._util import sign_align
for n, b, q, steps in [(64, 16, 1, 2), (100, 32, 2, 3), (130, 48, 0, 2), (300, 64, 1, 1), (200, 32, 2, 4), (520, 64, 2, 6)]:
    a = oracle.gaussian_matrix(n, n, 1000 + n)
    tg, ug, vg = _replay(a, b, q, 9, steps)
    tr, ur, vr = oracle.randutv(a, b=b, q=q, seed=9, max_steps=steps)
    d = sign_align(ug, ur)
    k = min(steps * b, n)
    print(json.dumps({"case": [n, b, q, steps], "cq": os.environ.get("RUTV_QR_CQ", "1"),
                      "t": float(np.max(np.abs(tg - d[:, None] * tr * d[None, :])) / np.linalg.norm(a)),
                      "diag_fin": float(np.max(np.abs(np.diag(tg)[:k] - np.diag(tr)[:k]) / np.abs(np.diag(tr)[:k]))),
                      "u": float(np.max(np.abs(ug - ur * d[None, :]))), "v": float(np.max(np.abs(vg - vr * d[None, :])))}), flush=True)
