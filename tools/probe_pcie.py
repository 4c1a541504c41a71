"""Host<->device copy bandwidth with exact-size pinned buffers: one stream vs several
concurrent streams (copy engines), H2D and D2H, and both directions at once."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2104_05782_b200 as rutv
GB = 8 * 1024 ** 3 // 8  # 8 GiB in doubles -> per-buffer elements below
n = 1 << 15  # 32768 x 32768 doubles = 8 GiB
h = rutv.PinnedMatrix(n, n)
h2 = rutv.PinnedMatrix(n, n)
d = torch.empty((n, n), dtype=torch.float64, device="cuda").T
d2 = torch.empty((n, n), dtype=torch.float64, device="cuda").T
out = {}
def run(tag, pairs, nstreams):
    ss = [torch.cuda.Stream() for _ in range(nstreams)]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k, (dst, src) in enumerate(pairs):
        cols = src.shape[1]
        per = (cols + nstreams - 1) // nstreams
        for j in range(nstreams):
            c0, c1 = j * per, min(cols, (j + 1) * per)
            if c0 < c1:
                rutv.copy_matrix_async(dst[:, c0:c1], src[:, c0:c1], ss[j].cuda_stream)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    gb = sum(8 * s.shape[0] * s.shape[1] for _, s in pairs) / 1e9
    out[tag] = round(gb / dt, 1)
for ns in (1, 2, 4):
    run(f"h2d_{ns}", [(d, h.array)], ns)
    run(f"d2h_{ns}", [(h.array, d)], ns)
run("both_2", [(d, h.array), (h2.array, d2)], 2)
print(json.dumps(out))
