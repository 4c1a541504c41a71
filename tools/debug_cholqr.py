"""Debug / timing: the Cholesky-QR2 fast path's small kernels and the full panel QR vs the oracle."""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, paper_2104_05782_b200 as rutv
from tests._util import cm_cuda, to_np
L = rutv.lib()
L.rutv_b200_debug_chol.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
L.rutv_b200_debug_lu.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
P = lambda t: C.c_void_p(t.data_ptr())
for s, p in ((2000, 128), (700, 100), (300, 37)):
    Y = oracle.gaussian_matrix(s, p, 3)
    G = Y.T @ Y
    Gd = cm_cuda(G); Rd = cm_cuda(np.zeros((p, p))); Ri = cm_cuda(np.zeros((p, p)))
    fl = L.rutv_b200_debug_chol(P(Gd), p, P(Rd), P(Ri))
    R1, R1i = to_np(Rd), to_np(Ri)
    print(s, p, "chol flag", fl, "err", np.max(np.abs(R1.T @ R1 - G)) / np.max(np.abs(G)), "inv err", np.max(np.abs(R1i @ R1 - np.eye(p))))
    Q = np.linalg.qr(Y)[0]
    Q = Q * np.sign(np.diag(np.linalg.qr(Y)[1]))[None, :]
    Qd = cm_cuda(Q); L1 = cm_cuda(np.zeros((p, p))); U = cm_cuda(np.zeros((p, p))); Ui = cm_cuda(np.zeros((p, p)))
    T = torch.zeros(p, dtype=torch.float64, device="cuda")
    fl = L.rutv_b200_debug_lu(P(Qd), s, p, P(L1), P(U), P(Ui), P(T))
    _, tau_ref, _ = oracle.hqr(Y)
    Lh = np.tril(to_np(L1), -1) + np.eye(p)
    Uh = Lh @ np.zeros((p, p))
    Bm = np.eye(p) - Q[:p]
    Ue = np.linalg.solve(Lh, Bm)
    print("   lu flag", fl, "tau err", np.max(np.abs(T.cpu().numpy() - tau_ref)), "Uinv err", np.max(np.abs(to_np(Ui) @ Ue - np.eye(p))),
          "LU err", np.max(np.abs(np.tril(Ue, -1))))
    # full panel QR through the C ABI
    A = cm_cuda(Y); tau = torch.zeros(p, dtype=torch.float64, device="cuda")
    L.rutv_b200_set_stream(C.c_uint64(torch.cuda.current_stream().cuda_stream))
    st = rutv.Status()
    L.rutv_b200_hqr_async(P(A), s, p, s, P(tau), C.byref(st))
    torch.cuda.synchronize()
    qr_ref, tau_ref, _ = oracle.hqr(Y)
    g = to_np(A)
    print("   panel: R err", np.max(np.abs(np.triu(g[:p]) - np.triu(qr_ref[:p]))) / np.max(np.abs(qr_ref)),
          "V err", np.max(np.abs(np.tril(g, -1) - np.tril(qr_ref, -1))), "tau err", np.max(np.abs(tau.cpu().numpy() - tau_ref)))
