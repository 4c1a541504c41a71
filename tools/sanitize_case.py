"""Small factorizations for compute-sanitizer runs (tests/test_gpu_sanitizer.py).

No torch: numpy + the C ABI only, so the sanitizer sees just this library's
kernels.  Covers the panel QR kernels (qr_reg by default, qr_cluster with
RUTV_QR_KERNEL=cluster), the batched cluster Jacobi (RUTV_JACOBI_CS forces the
cluster width), the grouped deferred beta stage (b <= 128), the rectangular
driver and the step API.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import paper_2104_05782_b200 as rutv  # noqa: E402

for (m, n, b, q) in [(160, 160, 32, 1), (200, 200, 64, 0), (130, 130, 128, 1), (90, 60, 16, 1)]:
    a = oracle.gaussian_matrix(m, n, 3 + m)
    t, u, v = rutv.factorize(a, b=b, q=q, seed=5)
    res = np.linalg.norm(a - u @ t @ v.T) / np.linalg.norm(a)
    assert res < 1e-12, (m, n, b, q, res)
a = oracle.gaussian_matrix(96, 96, 8)
qr, tau, twy = rutv.build_v_alpha(a, 24, 1, 1, 0)
p = np.asfortranarray(a[:, :24].copy())
rutv.build_u_alpha(p)
rutv.beta_stage(np.asfortranarray(a.copy()), 24)
print("sanitize case ok")
