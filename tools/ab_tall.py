"""A/B of the tall-panel Cholesky-QR2 path against the Householder kernels: time per panel and, with
`compare`, the difference of the packed results of two runs (RUTV_CHOLQR_MIN_ROWS=0 vs default).
  python tools/ab_tall.py run TAG [s,w ...]     -> /tmp/ab_tall_TAG_<s>_<w>.pt + one JSON line per shape
  python tools/ab_tall.py compare TAG1 TAG2 [s,w ...]"""
import ctypes as C, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

DEFAULT = [(50000, 512), (25000, 512), (10000, 512), (30000, 256), (15000, 256), (10000, 256), (8000, 128), (6144, 256)]


def shapes(args):
    return [tuple(int(x) for x in a.split(",")) for a in args] or DEFAULT


def run(tag, shp):
    import paper_2104_05782_b200 as rutv
    L = rutv.lib()
    L.rutv_b200_set_stream(C.c_uint64(torch.cuda.current_stream().cuda_stream))
    for s, w in shp:
        g = torch.Generator(device="cuda").manual_seed(s + w)
        x0 = torch.randn(w, s, dtype=torch.float64, device="cuda", generator=g).T
        xs = [x0.clone() for _ in range(4)]
        tau = torch.zeros(w, dtype=torch.float64, device="cuda")
        st = rutv.Status()
        call = lambda x: L.rutv_b200_hqr_async(C.c_void_p(x.data_ptr()), s, w, x.stride(1), C.c_void_p(tau.data_ptr()), C.byref(st))
        assert call(xs[0]) == 0, st.message
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for x in xs[1:]:
            call(x)
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        torch.save({"qr": xs[0].cpu(), "tau": tau.cpu()}, f"/tmp/ab_tall_{tag}_{s}_{w}.pt")
        print(json.dumps({"tag": tag, "s": s, "w": w, "ms": round(ms, 3), "us_per_col": round(ms * 1e3 / w, 2)}), flush=True)


def compare(t1, t2, shp):
    for s, w in shp:
        a, b = (torch.load(f"/tmp/ab_tall_{t}_{s}_{w}.pt") for t in (t1, t2))
        qa, qb = a["qr"], b["qr"]
        ra, rb = torch.triu(qa[:w]), torch.triu(qb[:w])
        va, vb = torch.tril(qa, -1), torch.tril(qb, -1)
        print(json.dumps({"s": s, "w": w, "r_rel": float((ra - rb).abs().max() / ra.abs().max()),
                          "v_abs": float((va - vb).abs().max()), "tau_abs": float((a["tau"] - b["tau"]).abs().max())}), flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(sys.argv[2], shapes(sys.argv[3:]))
    else:
        compare(sys.argv[2], sys.argv[3], shapes(sys.argv[4:]))
