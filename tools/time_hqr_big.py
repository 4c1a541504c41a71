"""Panel QR (hqr_panel + twy) time at the config-4/5 step shapes."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import ctypes as C
import paper_2104_05782_b200 as rutv
L = rutv.lib()
L.rutv_b200_set_stream(C.c_uint64(torch.cuda.current_stream().cuda_stream))
for s, w in [(50000, 512), (25000, 512), (10000, 512), (30000, 256), (15000, 256), (10000, 256), (4000, 128)]:
    xs = [torch.randn(w, s, dtype=torch.float64, device="cuda").T for _ in range(3)]
    tau = torch.zeros(w, dtype=torch.float64, device="cuda")
    st = rutv.Status()
    L.rutv_b200_hqr_async(C.c_void_p(xs[0].data_ptr()), s, w, s, C.c_void_p(tau.data_ptr()), C.byref(st))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for x in xs[1:]:
        L.rutv_b200_hqr_async(C.c_void_p(x.data_ptr()), s, w, s, C.c_void_p(tau.data_ptr()), C.byref(st))
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 2
    print(json.dumps({"s": s, "w": w, "ms": round(ms, 3), "us_per_col": round(ms * 1e3 / w, 2)}), flush=True)
