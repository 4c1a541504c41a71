"""Summarise ncu outputs into profiles/ (committed evidence).

  python tools/ncu_summary.py launches <launches.csv> <out.json>   # per-kernel shares of one factorization
  python tools/ncu_summary.py full <report.ncu-rep> <out.json>      # key --set full metrics per kernel
"""
import collections
import csv
import json
import subprocess
import sys


def launches(path, out):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, data = rows[0], rows[1:]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    marks = [i for i, r in enumerate(data) if "jacobi_kernel" in r[ki] or "jacobi_blk_kernel" in r[ki]]
    seg = data[marks[0] + 1: marks[1] + 1] if len(marks) >= 2 else data
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in seg:
        name = r[ki].split("(")[0]
        tot[name] += float(r[vi].replace(",", ""))
        cnt[name] += 1
    T = sum(tot.values())
    res = {"source": path, "note": "ncu gpu__time_duration.sum, --clock-control none; cold-cache, "
           "serialised launches of ONE factorization (between two batched-Jacobi launches): compare shares",
           "total_kernel_ms": T / 1e6, "launches": len(seg),
           "kernels": [{"name": k, "ms": v / 1e6, "share": v / T, "launches": cnt[k]}
                       for k, v in sorted(tot.items(), key=lambda x: -x[1])]}
    json.dump(res, open(out, "w"), indent=1)


def full(path, out):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr = rows[0]
    keys = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "launch__grid_size", "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active"]
    idx = {k: hdr.index(k) for k in keys if k in hdr}
    units = rows[1]
    kern = []
    for r in rows[2:]:
        kern.append({k: (r[i] + (" " + units[i] if units[i] else "")) for k, i in idx.items()})
    json.dump({"source": path, "kernels": kern}, open(out, "w"), indent=1)


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2], sys.argv[3])
