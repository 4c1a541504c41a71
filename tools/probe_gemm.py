"""GEMM throughput of the DMMA kernel on the randUTV step shapes (C ABI, incl. call overhead)."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2104_05782_b200 as rutv
from tests._util import cm_empty

def bench(M, N, K, ta, tb, beta=0.0, reps=10):
    a = cm_empty(*((K, M) if ta else (M, K))); b = cm_empty(*((N, K) if tb else (K, N))); c = cm_empty(M, N)
    torch.manual_seed(0); a.normal_(); b.normal_(); c.normal_()
    rutv.gemm(1.0, ta, a, tb, b, beta, c); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps): rutv.gemm(1.0, ta, a, tb, b, beta, c)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / reps
    print(json.dumps({"M": M, "N": N, "K": K, "ta": ta, "tb": tb, "ms": round(dt * 1e3, 3),
                      "tflops": round(2 * M * N * K / dt / 1e12, 2)}), flush=True)

for (M, N, K, ta, tb, beta) in [(8192, 8192, 8192, 0, 0, 0.0), (4000, 4000, 128, 0, 1, 1.0), (8000, 4000, 128, 0, 1, 1.0),
                                (4000, 3872, 128, 0, 0, 1.0), (4000, 128, 4000, 1, 0, 0.0), (4000, 128, 4000, 0, 0, 0.0),
                                (8000, 128, 4000, 0, 0, 0.0), (128, 3872, 4000, 1, 0, 0.0), (128, 128, 4000, 1, 0, 0.0),
                                (10000, 10000, 256, 0, 1, 1.0), (10000, 256, 10000, 1, 0, 0.0)]:
    bench(M, N, K, ta, tb, beta)
