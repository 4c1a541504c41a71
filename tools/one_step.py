"""First k steps of a BASELINE config (device-resident, in place) -- ncu target for the
large configs, where a whole factorization under ncu would take hours.
  python tools/one_step.py <config> <k> [warm=1]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2104_05782_b200 as rutv
import bench
cfg, k = int(sys.argv[1]), int(sys.argv[2])
warm = int(sys.argv[3]) if len(sys.argv) > 3 else 1
c = bench.CONFIGS[cfg]
n, b, q = c["n"], c["b"], c["q"]
a = torch.empty((n, n), dtype=torch.float64, device="cuda").T
bench.make_matrix(rutv, a, c["kind"], 1)
vt = torch.empty((n, 2 * n), dtype=torch.float64, device="cuda").T
u = torch.empty((n, n), dtype=torch.float64, device="cuda").T
for _ in range(warm + 1):
    rutv.factorize_device(a, vt[n:], u, vt[:n], b=b, q=q, seed=2, max_steps=k)
torch.cuda.synchronize()
print("ok", cfg, k)
