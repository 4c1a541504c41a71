"""Twy formation (hqr with twy) timing: kernel times of form_t at p = 256 / 512 (RUTV_FORMT=legacy for the single-CTA kernels)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from torch.profiler import ProfilerActivity, profile
import oracle, paper_2104_05782_b200 as rutv
from tests._util import cm_cuda, cm_empty, to_np
for s, p in ((2000, 256), (3000, 512), (1500, 384)):
    y = oracle.gaussian_matrix(s, p, 4)
    a0 = cm_cuda(y)
    tau = torch.zeros(p, dtype=torch.float64, device="cuda"); twy = cm_empty(p, p)
    a = a0.T.contiguous().T.clone(); rutv.hqr(a, tau, twy); torch.cuda.synchronize()
    _, _, twy_ref = oracle.hqr(y)
    err = float(np.max(np.abs(to_np(twy) - twy_ref)))
    a = cm_cuda(y)
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        rutv.hqr(a, tau, twy); torch.cuda.synchronize()
    ks = {}
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            k = ev.name.split("(")[0][-28:]
            ks[k] = round(ks.get(k, 0.0) + ev.device_time_total, 1)
    print(json.dumps({"s": s, "p": p, "mode": os.environ.get("RUTV_FORMT", "blocked"), "twy_err": err,
                      "form_t_us": {k: v for k, v in ks.items() if "form_t" in k}, "total_us": round(sum(ks.values()), 1)}), flush=True)
