"""Config-5 probe: in-place device factorization time, host-pointer (e2e) time,
pinned-allocation cost and HBM peak (nvidia-smi sampled)."""
import json
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2104_05782_b200 as rutv  # noqa: E402

n = int(os.environ.get("N", "50000"))
b = int(os.environ.get("B", "512"))
q = int(os.environ.get("Q", "2"))
smi = subprocess.Popen(["nvidia-smi", "--query-gpu=memory.used,clocks.sm,power.draw", "--format=csv,noheader,nounits",
                        "-lms", "500"], stdout=open("/tmp/smi_c5.csv", "w"))
out = {"n": n, "b": b, "q": q}
a = torch.empty((n, n), dtype=torch.float64, device="cuda").T
rutv.gaussian_matrix_device(a, 1)
vt = torch.empty((n, 2 * n), dtype=torch.float64, device="cuda").T
u = torch.empty((n, n), dtype=torch.float64, device="cuda").T
t, v = vt[n:, :], vt[:n, :]
torch.cuda.synchronize()
for rep in range(int(os.environ.get("REPS", "2"))):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rutv.factorize_device(a, t, u, v, b=b, q=q, seed=2, stream=torch.cuda.current_stream().cuda_stream)
    e1.record()
    torch.cuda.synchronize()
    out[f"device_s_{rep}"] = e0.elapsed_time(e1) / 1e3
    print(json.dumps(out), flush=True)
out["gflops"] = rutv.flops(n, b, q) / out["device_s_0"] / 1e9
d0 = torch.diagonal(t)[:4].cpu().numpy().tolist()
del vt, u, t, v
torch.cuda.synchronize()
torch.cuda.empty_cache()
if os.environ.get("E2E", "1") == "1":
    t0 = time.time()
    ha = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
    hs = [torch.empty((n, n), dtype=torch.float64, pin_memory=True) for _ in range(3)]
    out["pinned_alloc_s"] = time.time() - t0
    t0 = time.time()
    ha.copy_(a.T.cpu())
    out["stage_a_s"] = time.time() - t0
    del a
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    import ctypes as C
    o = rutv.make_opts(b=b, q=q, seed=2)
    st = rutv.Status()
    L = rutv.lib()
    for rep in range(int(os.environ.get("E2E_REPS", "1"))):
        t0 = time.time()
        L.rutv_b200_factorize(C.byref(o), C.c_void_p(ha.data_ptr()), n, n, n, None, 0,
                              C.c_void_p(hs[0].data_ptr()), n, C.c_void_p(hs[1].data_ptr()), n,
                              C.c_void_p(hs[2].data_ptr()), n, C.byref(st))
        rutv._raise(st)
        out[f"e2e_s_{rep}"] = time.time() - t0
        print(json.dumps(out), flush=True)
    out["diag_match"] = bool(torch.allclose(hs[0].T.diagonal()[:4], torch.tensor(d0, dtype=torch.float64)))
smi.terminate()
smi.wait()
rows = [ln.split(",") for ln in open("/tmp/smi_c5.csv") if ln.strip()]
out["hbm_peak_mib"] = max(float(r[0]) for r in rows)
out["sm_mhz_median"] = sorted(float(r[1]) for r in rows)[len(rows) // 2]
out["power_max_w"] = max(float(r[2]) for r in rows)
print(json.dumps(out), flush=True)
