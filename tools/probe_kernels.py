"""Time the QR and Jacobi kernels in isolation through the C ABI."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2104_05782_b200 as rutv
import oracle
from tests._util import cm_cuda, cm_empty

def tm(f, reps=5):
    f(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter(); f(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    return min(ts) * 1e3

for (m, n) in [(4000, 128), (2000, 128), (500, 128), (4000, 64), (10000, 256)]:
    a = cm_cuda(oracle.gaussian_matrix(m, n, 3))
    tau = torch.zeros(n, dtype=torch.float64, device="cuda")
    twy = cm_empty(n, n)
    def f():
        x = a.clone(memory_format=torch.contiguous_format) if False else a.T.contiguous().T
        rutv.hqr(x, tau, twy)
    print(json.dumps({"hqr": [m, n], "ms": round(tm(f), 3)}), flush=True)

for n in [16, 32, 64, 96, 112, 120, 128, 256]:
    g = oracle.gaussian_matrix(4 * n, n, 5)
    qr, _, _ = oracle.hqr(g)
    r = np.triu(qr[:n, :n])
    A = cm_cuda(r)
    U, V = cm_empty(n, n), cm_empty(n, n)
    s = torch.zeros(n, dtype=torch.float64, device="cuda")
    print(json.dumps({"svd_block": n, "ms": round(tm(lambda: rutv.svd_block(A, U, s, V)), 3)}), flush=True)
