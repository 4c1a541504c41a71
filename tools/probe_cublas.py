"""Reference point only (NOT the product): cuBLAS FP64 GEMM throughput on the same shapes
as tools/probe_gemm.py, via torch.matmul on float64 CUDA tensors.  Tells how far the
warp-level DMMA kernel is from NVIDIA's own sm_100 DGEMM on this chip."""
import json, time
import torch

def bench(M, N, K, ta, tb, beta, reps=10):
    a = torch.randn(M, K, dtype=torch.float64, device="cuda")
    b = torch.randn(K, N, dtype=torch.float64, device="cuda")
    c = torch.randn(M, N, dtype=torch.float64, device="cuda")
    f = (lambda: torch.addmm(c, a, b, beta=beta, alpha=1.0, out=c)) if beta else (lambda: torch.mm(a, b, out=c))
    f(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize()
    dt = e0.elapsed_time(e1) / 1e3 / reps
    print(json.dumps({"impl": "cublas", "M": M, "N": N, "K": K, "ms": round(dt * 1e3, 3),
                      "tflops": round(2 * M * N * K / dt / 1e12, 2)}), flush=True)

for (M, N, K, ta, tb, beta) in [(8192, 8192, 8192, 0, 0, 0.0), (16384, 16384, 4096, 0, 0, 0.0),
                                (4000, 4000, 128, 0, 1, 1.0), (8000, 4000, 128, 0, 1, 1.0),
                                (4000, 128, 4000, 1, 0, 0.0), (10000, 10000, 256, 0, 1, 1.0),
                                (50000, 50000, 512, 0, 0, 1.0), (50000, 512, 50000, 0, 0, 0.0)]:
    bench(M, N, K, ta, tb, beta)
