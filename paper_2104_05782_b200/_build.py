"""In-tree build of librutv_b200.so (nvcc, sm_100a only).

The shared library is the product: CUDA kernels + the C-ABI boundary
(include/rutv_b200.h).  It is built in place so it travels to the GPU box with
the repository snapshot.
"""
from __future__ import annotations

import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "librutv_b200.so")
OBJ = os.path.join(HERE, "_obj")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I", os.path.join(ROOT, "include"),
          "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills"]
# The device RNG restates the reference's no-contraction arithmetic
# (proj/CMakeLists.txt:17-18 -ffp-contract=off) -> no FMA fusion there.
PER_FILE = {"rng.cu": ["--fmad=false"]}
SOURCES = ["gemm_f64.cu", "rng.cu", "aux_kernels.cu", "qr_cluster.cu", "qr_reg.cu", "cholqr.cu", "jacobi.cu", "jacobi_blk.cu", "randutv.cu", "rect.cu", "grouped.cu", "gen.cu", "capi.cu", "stream_api.cu", "io_metrics.cu", "runtime.cu", "step_api.cu", "dist.cu"]


def _digest() -> str:
    h = hashlib.sha256()
    for name in sorted(os.listdir(CSRC)):
        with open(os.path.join(CSRC, name), "rb") as f:
            h.update(name.encode() + f.read())
    with open(os.path.join(ROOT, "include", "rutv_b200.h"), "rb") as f:
        h.update(f.read())
    h.update(" ".join(ARCH + COMMON).encode())
    return h.hexdigest()


def up_to_date() -> bool:
    stamp = LIB + ".sha256"
    return os.path.exists(LIB) and os.path.exists(stamp) and open(stamp).read().strip() == _digest()


def build(verbose: bool = False, force: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    os.makedirs(OBJ, exist_ok=True)
    objs = []
    procs = []
    for src in SOURCES:
        obj = os.path.join(OBJ, src.replace(".cu", ".o"))
        cmd = [NVCC, *ARCH, *COMMON, *PER_FILE.get(src, []), "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(obj)
    failed = []
    for src, p in procs:
        out = p.communicate()[0].decode()
        if p.returncode != 0:
            failed.append(f"--- {src}\n{out}")
        elif verbose and out.strip():
            print(out, file=sys.stderr)
    if failed:
        raise RuntimeError("nvcc failed:\n" + "\n".join(failed))
    tmp = LIB + ".tmp"
    # NCCL is dlopen'ed at first use by the sharded path (dist.cu), not linked: an
    # already-loaded libnccl.so.2 (torch's) must win over the system one
    subprocess.run([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart", "-ldl"], check=True)
    os.replace(tmp, LIB)
    with open(LIB + ".sha256", "w") as f:
        f.write(_digest())
    return LIB


if __name__ == "__main__":
    print(build(verbose=True, force="--force" in sys.argv))
