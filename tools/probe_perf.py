"""Quick perf probe: device-resident factorization timing + per-phase profile."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2104_05782_b200 as rutv

def cm(m, n):
    return torch.empty((n, m), dtype=torch.float64, device="cuda").T

def run(n, b, q, reps=int(os.environ.get('REPS', '3')), profile=os.environ.get('PROFILE', '1') == '1'):
    a = cm(n, n); rutv.normal_fill(1, 0, a)
    t, u, v = cm(n, n), cm(n, n), cm(n, n)
    rutv.factorize_device(a, t, u, v, b=b, q=q, seed=2)  # warm
    torch.cuda.synchronize()
    times = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); t0 = time.perf_counter()
        rutv.factorize_device(a, t, u, v, b=b, q=q, seed=2)
        torch.cuda.synchronize(); times.append(time.perf_counter() - t0)
    best = min(times)
    f = rutv.flops(n, b, q)
    out = {"n": n, "b": b, "q": q, "s": best, "gflops": f / best / 1e9}
    if profile:
        os.environ["RUTV_PROFILE"] = "1"
        rutv.factorize_device(a, t, u, v, b=b, q=q, seed=2)
        os.environ["RUTV_PROFILE"] = "0"
        out["phases_ms"] = {k: round(v, 3) for k, v in rutv.last_profile().items()}
        os.environ["RUTV_PROFILE"] = "2"  # critical-stream timeline with the overlap kept
        rutv.factorize_device(a, t, u, v, b=b, q=q, seed=2)
        os.environ["RUTV_PROFILE"] = "0"
        out["critical_ms"] = {k: round(v, 3) for k, v in rutv.last_profile().items()}
    print(json.dumps(out), flush=True)

for spec in sys.argv[1:]:
    n, b, q = (int(x) for x in spec.split(","))
    run(n, b, q)
