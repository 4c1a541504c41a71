"""Kernel-level GEMM timing through the asynchronous C ABI (no per-call host sync):
CUDA events around `reps` back-to-back launches on one stream.  Shapes of the randUTV step."""
import os, sys, json, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2104_05782_b200 as rutv
from tests._util import cm_empty

L = rutv.lib()
st = torch.cuda.current_stream()
L.rutv_b200_set_stream(C.c_uint64(st.cuda_stream))

def g(alpha, ta, a, tb, b, beta, c):
    s = rutv.Status()
    L.rutv_b200_gemm_async(C.c_double(alpha), ta, C.c_void_p(a.data_ptr()), a.shape[0], a.shape[1], a.stride(1),
                           tb, C.c_void_p(b.data_ptr()), b.shape[0], b.shape[1], b.stride(1), C.c_double(beta),
                           C.c_void_p(c.data_ptr()), c.shape[0], c.shape[1], c.stride(1), C.byref(s))
    assert s.code == 0, s.message

def bench(M, N, K, ta, tb, beta, reps=20):
    a = cm_empty(*((K, M) if ta else (M, K))); b = cm_empty(*((N, K) if tb else (K, N))); c = cm_empty(M, N)
    a.normal_(); b.normal_(); c.normal_()
    g(1.0, ta, a, tb, b, beta, c); torch.cuda.synchronize()
    reps = max(3, min(reps, int(2e12 / (2 * M * N * K))))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): g(1.0, ta, a, tb, b, beta, c)
    e1.record(); torch.cuda.synchronize()
    dt = e0.elapsed_time(e1) / 1e3 / reps
    out = {"M": M, "N": N, "K": K, "ta": ta, "tb": tb, "beta": beta, "us": round(dt * 1e6, 1),
           "tflops": round(2 * M * N * K / dt / 1e12, 2)}
    if dt < 2e-4:  # short calls: the ctypes loop is host-bound -- report CUPTI kernel time too
        from torch.profiler import profile, ProfilerActivity
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for _ in range(reps): g(1.0, ta, a, tb, b, beta, c)
            torch.cuda.synchronize()
        kt = sum(ev.device_time_total for ev in prof.events()
                 if ev.device_type == torch.autograd.DeviceType.CUDA) / reps / 1e6
        out["kernel_us"] = round(kt * 1e6, 1)
        out["kernel_tflops"] = round(2 * M * N * K / kt / 1e12, 2)
    return out

SHAPES = [(8192, 8192, 8192, 0, 0, 0.0), (4000, 4000, 128, 0, 1, 1.0), (8000, 4000, 128, 0, 1, 1.0),
          (4000, 3872, 128, 0, 0, 1.0), (2000, 2000, 128, 0, 1, 1.0), (4000, 128, 4000, 1, 0, 0.0),
          (4000, 128, 4000, 0, 0, 0.0), (8000, 128, 4000, 0, 0, 0.0), (128, 3872, 4000, 1, 0, 0.0),
          (2000, 128, 2000, 1, 0, 0.0), (10000, 10000, 256, 0, 1, 1.0), (10000, 256, 10000, 1, 0, 0.0),
          (20000, 20000, 512, 0, 1, 1.0), (20000, 512, 20000, 1, 0, 0.0),
          (128, 128, 4000, 1, 0, 0.0), (128, 128, 2000, 1, 0, 0.0), (4000, 128, 128, 0, 1, 0.0),
          (256, 256, 10000, 1, 0, 0.0), (512, 512, 50000, 1, 0, 0.0)]
if __name__ == "__main__":
    tag = sys.argv[1] if len(sys.argv) > 1 else ""
    bench(8192, 8192, 8192, 0, 0, 0.0, reps=30)  # warm the clocks up before measuring
    for sh in SHAPES:
        r = bench(*sh); r["tag"] = tag
        print(json.dumps(r), flush=True)
