"""Kernel list (CUPTI) of one config factorization, from the batched Jacobi on (the deferred beta stage)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile
import paper_2104_05782_b200 as rutv
n, b, q = (int(x) for x in (sys.argv[1:4] if len(sys.argv) > 3 else (4000, 128, 2)))
def cm(m, k): return torch.empty((k, m), dtype=torch.float64, device="cuda").T
a = cm(n, n); rutv.gaussian_matrix_device(a, 1)
t, u, v = cm(n, n), cm(n, n), cm(n, n)
rutv.factorize_device(a, t, u, v, b=b, q=q, seed=2)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    rutv.factorize_device(a, t, u, v, b=b, q=q, seed=2)
    torch.cuda.synchronize()
evs = sorted([e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA], key=lambda e: e.time_range.start)
idx = max(i for i, e in enumerate(evs) if "jacobi" in e.name)
t0 = evs[idx].time_range.start
for e in evs[idx:]:
    print(f"{(e.time_range.start - t0) / 1e3:9.3f} ms  {e.device_time_total:9.1f} us  {e.name[:80]}")
print("total from jacobi start to end:", (evs[-1].time_range.end - t0) / 1e3, "ms")
