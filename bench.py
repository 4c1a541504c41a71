#!/usr/bin/env python3
"""bench.py -- B200 blocked randUTV benchmark (BASELINE.json metric).

Metric: randUTV FP64 effective GFLOP/s = F(n, b, q) / time, F the reference's
algorithmic flop count (U and V built).
Workload (BASELINE.json configs[1]): n = 4000 geometric A = Q1 diag(sigma) Q2^T,
sigma_i = 10^(-12 (i-1)/(n-1)), b = 128, q = 2, full U, T, V.  A is built on
the device with the reference's Haar construction (metrics.cpp:95-110) from a
fixed seed -- synthetic data, no dataset involved.

A "step" is one complete factorization of that matrix.
  value : device-resident (A in HBM, outputs in HBM), CUDA events on the stream
          the library runs on, max over ranks.
  e2e   : the C-ABI host call rutv_b200_factorize with pinned host buffers:
          H2D of A and D2H of T, U, V inside the timed region.
Every input (A 128 MB, state 384 MB) exceeds the 126 MB L2, so no flush is
needed between iterations.

--impl reference: the reference's own CPU randUTV (oracle/_ref, compiled from
/root/reference/proj/src unmodified), single-threaded as the reference is by
contract, timed on a bounded sample of the same workload
family: n = 1000, b = 128, q = 2, geometric sigma 1 -> 1e-12.

--gpus N > 1 (torchrun): each rank factors its own matrix (independent
replicas, weak scaling); the 2D block-cyclic sharded path is not wired into
this bench yet.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_DEF, B_DEF, Q_DEF = 4000, 128, 2
SEED_A, SEED_G = 1, 2
DMMA_PEAK_TFLOPS = 37.1  # profiles/r01_dmma_peak.jsonl: mma.sync f64 burst, 148 SMs, 1.965 GHz
METRIC = "randUTV FP64 effective GFLOP/s & time at 1/2/4/8 B200; % of FP64 TC peak"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# BASELINE.json configs (seeds fixed here: A from SEED_A, the sketch stream from SEED_G)
CONFIGS = {
    1: dict(n=2000, b=128, q=0, kind="gaussian"),
    2: dict(n=4000, b=128, q=2, kind="geometric"),
    3: dict(n=10000, b=256, q=1, kind="gaussian"),
    4: dict(n=30000, b=256, q=2, kind="cliff"),
    5: dict(n=50000, b=512, q=2, kind="gaussian"),
}
KIND_TEXT = {"gaussian": "iid N(0,1)", "geometric": "geometric sigma 1->1e-12 (Haar product)",
             "cliff": "sigma=1 (i<=3000) then 1e-3*0.999^(i-3000) (Haar product)"}


def workload_name(n, b, q, kind="geometric", cfg=2):
    return f"config{cfg}: n={n} {KIND_TEXT[kind]}, b={b}, q={q}, full U/T/V"


def make_matrix(rutv, a, kind, seed):
    """A on the device with the reference's generators (metrics.cpp:90-110)."""
    n = a.shape[0]
    if kind == "gaussian":
        rutv.gaussian_matrix_device(a, seed)
    elif kind == "geometric":
        rutv.spectrum_matrix_device(a, seed, beta=10 ** (-12 / (n - 1)))
    else:
        import numpy as np
        i = np.arange(1, n + 1)
        sig = np.where(i <= 3000, 1.0, 1e-3 * 0.999 ** (i - 3000.0))
        rutv.spectrum_matrix_device(a, seed, sigma=sig)


# ----------------------------------------------------------------- clocks --
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.25)
        return self

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        rows = []
        try:
            for line in open(self.path):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 9:
                    rows.append(parts)
        except OSError:
            pass
        finally:
            try:
                os.unlink(self.path)
            except OSError:
                pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        smax = max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        loaded = [s for s in sm if s > 0.5 * smax] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": smax, "reasons": reasons,
                "samples": len(rows)}


# -------------------------------------------------------------- reference --
def reference_sample(n=1000, b=B_DEF, q=Q_DEF):
    """Time the unmodified reference randutv() (oracle/_ref) once on the sample (1 thread)."""
    import oracle
    a = oracle.geometric_matrix(n, n, 10 ** (-12 / (n - 1)), SEED_A, impl="ref")
    t0 = time.perf_counter()
    oracle.randutv(a, b=b, q=q, seed=SEED_G, impl="ref")
    dt = time.perf_counter() - t0
    return oracle.flops(n, b, q) / dt / 1e9, dt


def reference_ab_sample(n=2048, b=B_DEF, q=Q_DEF, workers=None):
    """The reference's multi-threaded algorithm-by-blocks driver (randutv_ab, every host
    thread) on the same family; it needs b | n, hence n = 2048 (16 x 128)."""
    import oracle
    workers = workers or os.cpu_count() or 1
    a = oracle.geometric_matrix(n, n, 10 ** (-12 / (n - 1)), SEED_A, impl="ref")
    t0 = time.perf_counter()
    oracle.ref_randutv_ab(a, b=b, q=q, seed=SEED_G, workers=workers)
    dt = time.perf_counter() - t0
    return oracle.flops(n, b, q) / dt / 1e9, dt, workers


def best_reference():
    """The faster of the reference's two CPU drivers on the box's host cores:
    (value GFLOP/s, seconds, cores, sample text)."""
    v1, dt1 = reference_sample(1000)
    try:
        v2, dt2, w = reference_ab_sample(2048)
    except Exception:  # the AB driver is an extra; the blocked one always exists
        v2, dt2, w = -1.0, 0.0, 1
    if v2 > v1:
        return v2, dt2, w, (f"reference randutv_ab (algorithm-by-blocks, {w} threads) on n=2048 of the config-2 "
                            f"family (b=128, q=2, geometric), {dt2:.2f} s; single-thread blocked randutv() on "
                            f"n=1000: {v1:.2f} GFLOP/s")
    return v1, dt1, 1, (f"reference randutv() (blocked, single thread by contract) on n=1000 of the config-2 "
                        f"family (b=128, q=2, geometric), {dt1:.2f} s")


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle
    if not oracle.available("ref"):
        kind = "port"
    else:
        kind = "reference"
    vals, times, cores, sample = [], [], 1, ""
    for i in range(args.warmup + args.steps):
        if kind == "reference":
            v, dt, cores, sample = best_reference()
        else:  # the C restatement (only if the reference library is missing)
            n = 1000
            a = oracle.geometric_matrix(n, n, 10 ** (-12 / (n - 1)), SEED_A)
            t0 = time.perf_counter()
            oracle.randutv(a, b=B_DEF, q=Q_DEF, seed=SEED_G)
            dt = time.perf_counter() - t0
            v = oracle.flops(n, B_DEF, Q_DEF) / dt / 1e9
            sample = f"C restatement of randutv() on n={n}, single thread"
        if i >= args.warmup:
            vals.append(v)
            times.append(dt)
    value = statistics.median(vals)
    sample += "; value = F(n,128,2)/t, median over the timed steps"
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "GFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1000 * statistics.median(times), 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(args.n, args.b, args.q, args.kind, args.config), "b": B_DEF,
                   "q": Q_DEF, "parallelism": f"cpu-{cores}threads"},
        "cpu_baseline": {"value": round(value, 4), "unit": "GFLOP/s", "cores": cores, "kind": kind,
                         "sample": sample},
        "e2e": {"value": round(value, 4), "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ------------------------------------------------------------------- B200 --
def cm(torch, m, n, dev):
    return torch.empty((n, m), dtype=torch.float64, device=dev).T


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=2, choices=sorted(CONFIGS),
                    help="BASELINE.json config (default 2, the single-GPU headline)")
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--b", type=int, default=None)
    ap.add_argument("--q", type=int, default=None)
    ap.add_argument("--sharded", action="store_true",
                    help="N > 1: ONE matrix on the 2D block-cyclic grid (dist.py, NCCL), strong scaling; "
                         "default: one independent factorization per GPU (weak scaling)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 0)
    cfgd = CONFIGS[args.config]
    args.n = cfgd["n"] if args.n is None else args.n
    args.b = cfgd["b"] if args.b is None else args.b
    args.q = cfgd["q"] if args.q is None else args.q
    args.kind = cfgd["kind"]
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    import paper_2104_05782_b200 as rutv

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    n, b, q = args.n, args.b, args.q
    F = rutv.flops(n, b, q)
    if args.sharded:
        return run_sharded(args, torch, dist, rutv, world, rank, local, dev, F)

    a = cm(torch, n, n, dev)
    make_matrix(rutv, a, args.kind, SEED_A + rank)
    t, u, v = cm(torch, n, n, dev), cm(torch, n, n, dev), cm(torch, n, n, dev)
    stream = torch.cuda.current_stream(dev)
    sh = stream.cuda_stream

    def step():
        rutv.factorize_device(a, t, u, v, b=b, q=q, seed=SEED_G, stream=sh)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    launches0 = rutv.launch_count()
    with ClockSampler(local) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    launches = rutv.launch_count() - launches0
    ms = e0.elapsed_time(e1) / args.steps
    clocks = clk.summary()
    ms_t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    value = world * F / (ms_max / 1e3) / 1e9

    # ---- e2e through the C ABI with pinned host buffers
    e2e = None
    if not args.no_e2e:
        import ctypes as C
        import numpy as np
        ha = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
        ha.copy_(a.T.cpu())  # column-major bytes of A
        ht = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
        hu = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
        hv = torch.empty((n, n), dtype=torch.float64, pin_memory=True)
        o = rutv.make_opts(b=b, q=q, seed=SEED_G, device=local, stream=sh)
        st = rutv.Status()
        L = rutv.lib()

        def e2e_step():
            L.rutv_b200_factorize(C.byref(o), C.c_void_p(ha.data_ptr()), n, n, n, None, 0,
                                  C.c_void_p(ht.data_ptr()), n, C.c_void_p(hu.data_ptr()), n,
                                  C.c_void_p(hv.data_ptr()), n, C.byref(st))
            rutv._raise(st)

        e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.steps):
            e2e_step()
        f1.record(stream)
        torch.cuda.synchronize()
        ems = torch.tensor([f0.elapsed_time(f1) / args.steps], device=dev)
        if world > 1:
            dist.all_reduce(ems, op=dist.ReduceOp.MAX)
        e2e = {"value": round(world * F / (float(ems.item()) / 1e3) / 1e9, 3), "unit": "GFLOP/s",
               "ms_per_step": round(float(ems.item()), 3),
               "h2d_bytes_per_step": 8 * n * n, "d2h_bytes_per_step": 3 * 8 * n * n}
        # sanity: the host result matches the device one (same stream of deviates)
        assert np.allclose(ht.numpy().T[:4, :4], t.cpu().numpy()[:4, :4])

    # ---- roofline of the dominant kernel (DMMA GEMM), separate profiled pass
    # Streams serialized (RUTV_OVERLAP=0) so each GEMM's event bracket is its own
    # launch time, not time shared with concurrent kernels of the other streams.
    os.environ["RUTV_GEMM_PROFILE"] = "1"
    os.environ["RUTV_OVERLAP"] = "0"
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    step()
    p1.record(stream)
    torch.cuda.synchronize()
    pass_ms = p0.elapsed_time(p1)
    os.environ["RUTV_GEMM_PROFILE"] = "0"
    os.environ["RUTV_OVERLAP"] = "1"
    gp = rutv.gemm_profile()
    gemm_tflops = gp["flops"] / (gp["ms"] / 1e3) / 1e12 if gp["ms"] > 0 else None
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "gemm_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get("bytes_per_launch")
        except (OSError, ValueError):
            traffic = None
    roofline = {"bound": "tensor", "achieved": round(gemm_tflops, 3) if gemm_tflops else None,
                "peak": DMMA_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": round(gemm_tflops / DMMA_PEAK_TFLOPS, 4) if gemm_tflops else None,
                "traffic": traffic, "kernel": "dgemm_kernel (+split-K reduce)",
                "gemm_ms_per_step": round(gp["ms"], 3), "gemm_launches": gp["launches"],
                "gemm_share_of_serialized_step": round(gp["ms"] / pass_ms, 4) if pass_ms > 0 else None,
                "serialized_step_ms": round(pass_ms, 3),
                "step_frac_of_peak": round(F / (ms / 1e3) / 1e12 / DMMA_PEAK_TFLOPS, 4),
                "peak_source": "measured DMMA burst (profiles/r01_dmma_peak.jsonl); "
                               "MEASURED_PEAKS.json has no FP64 entry"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            import oracle
            if oracle.available("ref"):
                v_ref, dt, cores, sample = best_reference()
                cpu = {"value": round(v_ref, 4), "unit": "GFLOP/s", "cores": cores, "kind": "reference",
                       "sample": sample}
        except Exception as exc:  # the baseline is reported, never required
            cpu = {"value": None, "unit": "GFLOP/s", "cores": 1, "kind": "reference",
                   "sample": f"unavailable: {exc}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_max, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": f"synthetic (device-generated {KIND_TEXT[args.kind]}, seed {SEED_A})",
            "config": {"workload": workload_name(n, b, q, args.kind, args.config), "n": n, "b": b, "q": q,
                       "flops_per_step": F, "parallelism": "replicas" if world > 1 else "single",
                       "l2": "inputs (A 128 MB + 384 MB state) exceed the 126 MB L2; no flush"},
            "e2e": e2e, "gpu_launches": launches, "clocks": clocks, "roofline": roofline,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


# ---------------------------------------------------------- sharded (2D) --
def run_sharded(args, torch, dist, rutv, world, rank, local, dev, F):
    """ONE matrix on the P x Q block-cyclic grid (dist.py): strong scaling.
    value = F / (max over ranks of the device time of one factorization)."""
    from paper_2104_05782_b200.dist import CudaOps, Grid, factorize_dist, grid_shape, make_comms, scatter_grid
    n, b, q = args.n, args.b, args.q
    P, Q = grid_shape(world)
    grid = Grid(n, b, P, Q, rank)
    comms = make_comms(grid) if world > 1 else None
    full = cm(torch, n, n, dev)
    make_matrix(rutv, full, args.kind, SEED_A)  # same matrix on every rank (deterministic generator)
    a_loc = scatter_grid(full, grid)
    del full
    torch.cuda.empty_cache()
    ops = CudaOps(dev)
    stream = torch.cuda.current_stream(dev)

    def step(x):
        return factorize_dist(x, grid, q=q, seed=SEED_G, ops=ops, comms=comms)

    for _ in range(args.warmup):
        step(a_loc)
    torch.cuda.synchronize()
    launches0 = rutv.launch_count()
    with ClockSampler(local) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            step(a_loc)
        e1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    launches = rutv.launch_count() - launches0
    ms_t = torch.tensor([e0.elapsed_time(e1) / args.steps], device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())
    # e2e: this rank's blocks from pinned host memory, results back to pinned host memory
    e2e = None
    if not args.no_e2e:
        mr, mc = a_loc.shape
        ha = torch.empty((mc, mr), dtype=torch.float64, pin_memory=True).T
        ha.copy_(a_loc)
        hout = [torch.empty((mc, mr), dtype=torch.float64, pin_memory=True).T for _ in range(3)]
        dbuf = torch.empty_like(a_loc)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.steps):
            dbuf.copy_(ha, non_blocking=True)
            t, u, v = step(dbuf)
            for h, d in zip(hout, (t, u, v)):
                h.copy_(d, non_blocking=True)
        f1.record(stream)
        torch.cuda.synchronize()
        ems = torch.tensor([f0.elapsed_time(f1) / args.steps], device=dev)
        if world > 1:
            dist.all_reduce(ems, op=dist.ReduceOp.MAX)
        e2e = {"value": round(F / (float(ems.item()) / 1e3) / 1e9, 3), "unit": "GFLOP/s",
               "ms_per_step": round(float(ems.item()), 3),
               "h2d_bytes_per_step": 8 * mr * mc, "d2h_bytes_per_step": 3 * 8 * mr * mc, "per_rank": True}
    if rank == 0:
        value = F / (ms / 1e3) / 1e9
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": f"synthetic (device-generated {KIND_TEXT[args.kind]}, seed {SEED_A})",
            "config": {"workload": workload_name(n, b, q, args.kind, args.config), "n": n, "b": b, "q": q,
                       "flops_per_step": F, "parallelism": f"2d-block-cyclic {P}x{Q}",
                       "l2": "state exceeds the 126 MB L2; no flush"},
            "e2e": e2e, "gpu_launches": launches, "clocks": clk.summary(),
            "roofline": {"bound": "tensor", "achieved": round(value / 1e3 / world, 3), "peak": DMMA_PEAK_TFLOPS,
                         "unit": "TFLOP/s", "frac": round(value / 1e3 / world / DMMA_PEAK_TFLOPS, 4),
                         "traffic": None, "kernel": "whole factorization per GPU (dist driver)"},
            "cpu_baseline": None,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
