"""Config-5 host-pointer call (rutv_b200_factorize) timing with the library pool trimmed
after every call (default) vs kept (RUTV_POOL_KEEP_MB large): the allocation share of e2e."""
import ctypes as C, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2104_05782_b200 as rutv
n, b, q = 50000, 512, 2
ha = rutv.PinnedMatrix(n, n)
a = torch.empty((n, n), dtype=torch.float64, device="cuda").T
rutv.gaussian_matrix_device(a, 1)
rutv.copy_matrix_async(ha.array, a, 0)
torch.cuda.synchronize()
del a
torch.cuda.empty_cache()
hout = [rutv.PinnedMatrix(n, n) for _ in range(3)]
o = rutv.make_opts(b=b, q=q, seed=2)
st = rutv.Status()
L = rutv.lib()
out = {"keep_mb": os.environ.get("RUTV_POOL_KEEP_MB", "default")}
for rep in range(int(os.environ.get("REPS", "2"))):
    t0 = time.perf_counter()
    L.rutv_b200_factorize(C.byref(o), ha.ptr, n, n, n, None, 0, hout[0].ptr, n, hout[1].ptr, n, hout[2].ptr, n,
                          C.byref(st))
    rutv._raise(st)
    out[f"s_{rep}"] = round(time.perf_counter() - t0, 3)
    print(json.dumps(out), flush=True)
