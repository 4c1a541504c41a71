"""One device-resident factorization (after one warm-up) -- ncu launch-list target."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2104_05782_b200 as rutv
n, b, q = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (4000, 128, 2)))
def cm(m, k): return torch.empty((k, m), dtype=torch.float64, device="cuda").T
a = cm(n, n); rutv.gaussian_matrix_device(a, 1)
t, u, v = cm(n, n), cm(n, n), cm(n, n)
for _ in range(2):
    rutv.factorize_device(a, t, u, v, b=b, q=q, seed=2)
torch.cuda.synchronize()
print("ok", n, b, q)
