"""Short-K update shapes (configs 1-3): 128x64 vs 64x64 tiles (RUTV_GEMM_PLAN=1)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tools.gemm_bench import bench
bench(8192, 8192, 8192, 0, 0, 0.0, reps=10)
for sh in [(4000, 4000, 128, 0, 1, 1.0), (3872, 3872, 128, 0, 1, 1.0), (2000, 2000, 128, 0, 1, 1.0),
           (8000, 4000, 128, 0, 1, 1.0), (4000, 3872, 128, 0, 0, 1.0), (10000, 10000, 256, 0, 1, 1.0),
           (6000, 6000, 256, 0, 1, 1.0), (2000, 1872, 128, 1, 0, 1.0)]:
    r = bench(*sh)
    r["plan"] = os.environ.get("RUTV_GEMM_PLAN", "0")
    print(json.dumps(r), flush=True)
