"""Kernel time of the Jacobi SVD (svd_block) on R factors of Gaussian panels, n in argv."""
import json
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from torch.profiler import ProfilerActivity, profile
import oracle
import paper_2104_05782_b200 as rutv
from tests._util import cm_cuda, cm_empty

for n in [int(x) for x in sys.argv[1:]] or [128, 256, 512]:
    qr, _, _ = oracle.hqr(oracle.gaussian_matrix(4 * n, n, 5))
    A = cm_cuda(np.triu(qr[:n, :n]))
    U, V = cm_empty(n, n), cm_empty(n, n)
    s = torch.zeros(n, dtype=torch.float64, device="cuda")
    rutv.svd_block(A, U, s, V)
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        rutv.svd_block(A, U, s, V)
        torch.cuda.synchronize()
    ks = {}
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            ks[ev.name.split("(")[0][-40:]] = ks.get(ev.name.split("(")[0][-40:], 0.0) + ev.device_time_total
    print(json.dumps({"n": n, "kernels_us": {k: round(v, 1) for k, v in ks.items()}}), flush=True)
