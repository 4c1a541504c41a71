"""Config-5 step GEMM shapes: our DMMA kernel (raster on / off) vs cuBLAS (reference point)."""
import json, os, sys, subprocess
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
SHAPES = [  # (M, N, K, ta, tb, beta)
    (50000, 50000, 512, 0, 1, 1.0),   # rank-512 update  X -= Zx M'
    (50000, 512, 50000, 1, 0, 0.0),   # sketch Y = T22' G / projection W'B (TN)
    (50000, 512, 50000, 0, 0, 0.0),   # Z = T22 Y, Zx = X W (NN)
    (512, 49488, 50000, 1, 0, 0.0),   # Zl = W_u' B (TN, M = b)
    (100000, 512, 50000, 0, 0, 0.0),  # [V; T] W (NN, 2n rows)
    (30000, 30000, 256, 0, 1, 1.0),   # config 4 update
    (30000, 256, 30000, 1, 0, 0.0),   # config 4 sketch
    (8192, 8192, 8192, 0, 0, 0.0),
]
if __name__ == "__main__":
    import torch
    import paper_2104_05782_b200 as rutv
    from tools.gemm_bench import bench
    bench(8192, 8192, 8192, 0, 0, 0.0, reps=20)
    for sh in SHAPES:
        r = bench(*sh, reps=5)
        r["raster"] = os.environ.get("RUTV_GEMM_RASTER", "1")
        print(json.dumps(r), flush=True)
