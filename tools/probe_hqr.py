"""One hqr of an s x w Gaussian panel through the C ABI (ncu target)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2104_05782_b200 as rutv
import oracle
from tests._util import cm_cuda, cm_empty
s, w = (int(sys.argv[1]), int(sys.argv[2])) if len(sys.argv) > 2 else (2000, 128)
a = cm_cuda(oracle.gaussian_matrix(s, w, 3))
tau = torch.zeros(w, dtype=torch.float64, device="cuda")
twy = cm_empty(w, w)
for _ in range(2):
    x = a.T.contiguous().T
    rutv.hqr(x, tau, twy)
torch.cuda.synchronize()
print("ok")
