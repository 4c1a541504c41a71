"""Phase clocks of the Cholesky-QR2 small-factorization kernels (cqr_chol / cqr_lu) on one panel."""
import ctypes as C, os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2104_05782_b200 as rutv
L = rutv.lib()
L.rutv_b200_set_stream(C.c_uint64(torch.cuda.current_stream().cuda_stream))
os.environ["RUTV_CHOLQR"] = "1"
s, p = (int(x) for x in (sys.argv[1:] or ["2000", "128"]))
for rep in range(3):
    a = torch.randn(p, s, dtype=torch.float64, device="cuda").T
    tau = torch.zeros(p, dtype=torch.float64, device="cuda")
    st = rutv.Status()
    L.rutv_b200_hqr_async(C.c_void_p(a.data_ptr()), s, p, s, C.c_void_p(tau.data_ptr()), C.byref(st))
    torch.cuda.synchronize()
clk = (C.c_longlong * 128)()
L.rutv_b200_debug_cqr_clocks(clk)
c = list(clk)
out = {}
for name, b in (("chol1", 0), ("chol2", 16), ("lu", 32)):
    out[name] = [c[b + i] - c[b] if c[b + i] else None for i in range(17)]
out['chol1_diag0'] = [c[60 + i] - c[1] for i in range(4)]
print(json.dumps(out))
