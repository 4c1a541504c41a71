"""One GEMM launch of a given shape: ours (C ABI) or cuBLAS (torch) -- ncu target."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
impl, M, N, K, beta = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), float(sys.argv[5])
ta = int(sys.argv[6]) if len(sys.argv) > 6 else 0
tb = int(sys.argv[7]) if len(sys.argv) > 7 else 0
if impl == "cublas":
    a = torch.randn(M, K, dtype=torch.float64, device="cuda"); b = torch.randn(K, N, dtype=torch.float64, device="cuda")
    c = torch.randn(M, N, dtype=torch.float64, device="cuda")
    for _ in range(2):
        torch.addmm(c, a, b, beta=beta, out=c) if beta else torch.mm(a, b, out=c)
else:
    import paper_2104_05782_b200 as rutv
    from tests._util import cm_empty
    a = cm_empty(K, M) if ta else cm_empty(M, K)
    b = cm_empty(N, K) if tb else cm_empty(K, N)
    c = cm_empty(M, N)
    a.normal_(); b.normal_(); c.normal_()
    for _ in range(2):
        rutv.gemm(1.0, ta, a, tb, b, beta, c)
torch.cuda.synchronize()
