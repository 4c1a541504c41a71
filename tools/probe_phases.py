"""Critical-stream phase timeline (RUTV_PROFILE=2) and serialized phase profile (=1) of the
first k steps of a BASELINE config: where a step's time goes at large n."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2104_05782_b200 as rutv
import bench

cfg, k = int(sys.argv[1]), int(sys.argv[2])
c = bench.CONFIGS[cfg]
n, b, q = c["n"], c["b"], c["q"]
a = torch.empty((n, n), dtype=torch.float64, device="cuda").T
bench.make_matrix(rutv, a, c["kind"], 1)
vt = torch.empty((n, 2 * n), dtype=torch.float64, device="cuda").T
u = torch.empty((n, n), dtype=torch.float64, device="cuda").T
t, v = vt[n:], vt[:n]
out = {"config": cfg, "steps": k}
for mode in ("0", "2", "1"):
    os.environ["RUTV_PROFILE"] = mode
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rutv.factorize_device(a, t, u, v, b=b, q=q, seed=2, max_steps=k)
    e1.record()
    torch.cuda.synchronize()
    out[f"ms_mode{mode}"] = round(e0.elapsed_time(e1), 2)
    if mode != "0":
        out[f"phases_mode{mode}"] = {kk: round(vv, 2) for kk, vv in rutv.last_profile().items()}
os.environ["RUTV_PROFILE"] = "0"
print(json.dumps(out), flush=True)
