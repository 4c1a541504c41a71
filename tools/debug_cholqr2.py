import ctypes as C, os, sys
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import oracle, paper_2104_05782_b200 as rutv
from tests._util import to_np
L = rutv.lib()
L.rutv_b200_set_stream(C.c_uint64(torch.cuda.current_stream().cuda_stream))
s, w = 2000, 128
torch.manual_seed(0)
a0 = torch.randn(w, s, dtype=torch.float64, device="cuda").T
xs = [a0.T.contiguous().T for _ in range(4)]
Y = to_np(a0)
qr_ref, tau_ref, _ = oracle.hqr(Y)
tau = torch.zeros(w, dtype=torch.float64, device="cuda")
for i, x in enumerate(xs):
    st = rutv.Status()
    L.rutv_b200_hqr_async(C.c_void_p(x.data_ptr()), x.shape[0], x.shape[1], x.stride(1), C.c_void_p(tau.data_ptr()), C.byref(st))
    torch.cuda.synchronize()
    print(i, "tau err", np.max(np.abs(tau.cpu().numpy() - tau_ref)),
          "other panels changed:", [float((xx - a0).abs().max()) for xx in xs[i + 1:]],
          "a0 changed:", float((a0 - torch.from_numpy(Y).cuda()).abs().max()), flush=True)
