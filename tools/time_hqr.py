"""Time rutv.hqr (cluster Householder panel QR) over panel shapes: us per call and per column."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import ctypes as C
import paper_2104_05782_b200 as rutv

L = rutv.lib()
L.rutv_b200_set_stream(C.c_uint64(torch.cuda.current_stream().cuda_stream))


def hqr(x, tau):
    st = rutv.Status()
    rc = L.rutv_b200_hqr_async(C.c_void_p(x.data_ptr()), x.shape[0], x.shape[1], x.stride(1),
                               C.c_void_p(tau.data_ptr()), C.byref(st))
    assert rc == 0, st.message

shapes = [tuple(int(x) for x in s.split(",")) for s in sys.argv[1:]] or [
    (128, 128), (256, 128), (512, 128), (1000, 128), (2000, 128), (3000, 128), (4000, 128), (10000, 256)]
for s, w in shapes:
    a0 = torch.randn(w, s, dtype=torch.float64, device="cuda").T
    tau = torch.zeros(w, dtype=torch.float64, device="cuda")
    xs = [a0.clone() for _ in range(6)]  # distinct panels (each call factors in place)
    hqr(xs[0], tau)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for x in xs[1:]:
        hqr(x, tau)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / 5
    # device-side kernel time (CUPTI through torch.profiler)
    from torch.profiler import profile, ProfilerActivity
    xs = [a0.clone() for _ in range(6)]  # fresh panels again for the profiled pass
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for x in xs[1:]:
            hqr(x, tau)
        torch.cuda.synchronize()
    kt = {}
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            kt[ev.name[:40]] = kt.get(ev.name[:40], 0.0) + ev.device_time_total / 5
    kus = sum(kt.values())
    print(json.dumps({"s": s, "w": w, "us": round(us, 1), "kernel_us": round(kus, 1),
                      "us_per_col": round(kus / w, 2), "kernels": {k: round(v, 1) for k, v in kt.items()}}), flush=True)
