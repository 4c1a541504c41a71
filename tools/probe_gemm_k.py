"""Kernel-only GEMM times (CUPTI via torch.profiler) on the randUTV step shapes, async C ABI."""
import ctypes as C
import json
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from torch.profiler import ProfilerActivity, profile
import paper_2104_05782_b200 as rutv

L = rutv.lib()
L.rutv_b200_set_stream(C.c_uint64(torch.cuda.current_stream().cuda_stream))


def cm(m, n):
    return torch.randn(n, m, dtype=torch.float64, device="cuda").T


def gemm(alpha, ta, a, tb, b, beta, c):
    st = rutv.Status()
    rc = L.rutv_b200_gemm_async(alpha, ta, C.c_void_p(a.data_ptr()), a.shape[0], a.shape[1], a.stride(1), tb,
                                C.c_void_p(b.data_ptr()), b.shape[0], b.shape[1], b.stride(1), beta,
                                C.c_void_p(c.data_ptr()), c.shape[0], c.shape[1], c.stride(1), C.byref(st))
    assert rc == 0, st.message


shapes = [(4000, 128, 4000, 1, 0, 0.0), (4000, 128, 4000, 0, 0, 0.0), (2000, 128, 2000, 1, 0, 0.0),
          (4000, 4000, 128, 0, 1, 1.0), (4000, 3872, 128, 0, 0, 1.0), (2000, 2000, 128, 0, 1, 1.0),
          (128, 3872, 4000, 1, 0, 0.0), (128, 128, 4000, 1, 0, 0.0), (4000, 128, 128, 0, 1, 0.0),
          (8192, 8192, 8192, 0, 0, 0.0), (10000, 256, 10000, 1, 0, 0.0), (10000, 10000, 256, 0, 1, 1.0)]
if len(sys.argv) > 1:
    shapes = [tuple(float(x) if i == 5 else int(x) for i, x in enumerate(s.split(","))) for s in sys.argv[1:]]
for (M, N, K, ta, tb, beta) in shapes:
    a = cm(K, M) if ta else cm(M, K)
    b = cm(N, K) if tb else cm(K, N)
    c = cm(M, N)
    for _ in range(2):
        gemm(1.0, ta, a, tb, b, beta, c)
    torch.cuda.synchronize()
    reps = 5
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(reps):
            gemm(1.0, ta, a, tb, b, beta, c)
        torch.cuda.synchronize()
    ks = {}
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            ks[ev.name.split("(")[0][-60:]] = ks.get(ev.name.split("(")[0][-60:], 0.0) + ev.device_time_total / reps
    us = sum(ks.values())
    print(json.dumps({"M": M, "N": N, "K": K, "ta": ta, "tb": tb, "beta": beta, "kernel_us": round(us, 1),
                      "tflops": round(2 * M * N * K / us / 1e6, 2),
                      "kernels": {k: round(v, 1) for k, v in ks.items()}}), flush=True)
