"""profiles/gemm_traffic.json (bench.py's roofline.traffic) from an ncu --set full summary
made by tools/ncu_summary.py: mean dram__bytes_read + dram__bytes_write per GEMM launch,
and per tile class.

  python tools/traffic_json.py <gemm_full summary.json> <source note> [out]
"""
import collections
import json
import re
import sys

SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def val(s):
    v, u = s.split()[:2] if len(s.split()) > 1 else (s, "byte")
    return float(v.replace(",", "")) * SCALE.get(u, 1.0)


def pct(s):
    return float(s.split()[0].replace(",", ""))


def us(s):
    v, u = s.split()[:2]
    return float(v.replace(",", "")) * {"ns": 1e-3, "us": 1.0, "ms": 1e3}[u]


src, note = sys.argv[1], sys.argv[2]
out = sys.argv[3] if len(sys.argv) > 3 else "profiles/gemm_traffic.json"
ks = json.load(open(src))["kernels"]
cls = collections.defaultdict(list)
for k in ks:
    cls[re.sub(r"^void ", "", k["Kernel Name"]).split("(")[0]].append(k)
tot = [val(k["dram__bytes_read.sum"]) + val(k["dram__bytes_write.sum"]) for k in ks]
res = {"source": note, "launches_sampled": len(ks), "bytes_per_launch": sum(tot) / len(tot), "classes": {}}
for name, v in cls.items():
    res["classes"][name] = {
        "launches": len(v),
        "dram_MB_per_launch": round(sum(val(k["dram__bytes_read.sum"]) + val(k["dram__bytes_write.sum"]) for k in v) / len(v) / 1e6, 2),
        "us_per_launch": round(sum(us(k["gpu__time_duration.sum"]) for k in v) / len(v), 1),
        "dmma_active_pct": round(sum(pct(k["sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active"]) for k in v) / len(v), 1),
    }
json.dump(res, open(out, "w"), indent=1)
print(json.dumps({"bytes_per_launch": res["bytes_per_launch"], "classes": len(res["classes"])}))
