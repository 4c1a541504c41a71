"""One 128x128 Jacobi SVD through the C ABI (ncu target)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2104_05782_b200 as rutv
import oracle
from tests._util import cm_cuda, cm_empty
n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
qr, _, _ = oracle.hqr(oracle.gaussian_matrix(4 * n, n, 5))
A = cm_cuda(np.triu(qr[:n, :n]))
U, V = cm_empty(n, n), cm_empty(n, n)
s = torch.zeros(n, dtype=torch.float64, device="cuda")
for _ in range(2):
    rutv.svd_block(A, U, s, V)
torch.cuda.synchronize()
print("ok", float(s[0]))
