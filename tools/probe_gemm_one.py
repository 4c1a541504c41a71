import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2104_05782_b200 as rutv
from tests._util import cm_empty
M, N, K, ta, tb, beta = (int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5]), float(sys.argv[6]))
a = cm_empty(*((K, M) if ta else (M, K))); b = cm_empty(*((N, K) if tb else (K, N))); c = cm_empty(M, N)
a.normal_(); b.normal_(); c.normal_()
for _ in range(2): rutv.gemm(1.0, ta, a, tb, b, beta, c)
torch.cuda.synchronize(); print("ok")
