#!/usr/bin/env python3
"""bench.py -- B200 blocked randUTV benchmark (BASELINE.json metric).

Metric: randUTV FP64 effective GFLOP/s = F(n, b, q) / time, F the reference's
algorithmic flop count (U and V built).

Workload (default): BASELINE.json configs[4] -- "config 5", the largest
single-GPU configuration and the north-star target: n = 50000 iid N(0,1) A
(gaussian_matrix, metrics.cpp:90-93, generated on the device from seed 1),
b = 512, q = 2, full U, T, V.  `--config 1..4` selects the other BASELINE
configs (they are parity-test cases, tests/test_gpu_configs.py).  Synthetic
data, no dataset involved.

A "step" is one complete factorization of that matrix.
  value : device-resident: A and the outputs in HBM (T and V stacked in one
          buffer, U separate -- factored in place, 4 n^2 doubles = 80 GB at
          config 5), CUDA events on the stream the library runs on, max over ranks.
  e2e   : the reference-facing C-ABI host call rutv_b200_factorize with pinned
          host buffers: H2D of A and D2H of T, U, V inside the timed region.
          At n >= 20000 it is timed over min(K, --e2e-steps) steps (default 2),
          after one untimed call: one config-5 call is ~43 s and the driver's arm
          has 1800 s.  The call keeps its device workspace cached between calls
          (rutv_opts.keep_workspace, as a caller factoring repeatedly would).
Every input exceeds the 126 MB L2 (config 5: 20 GB A, 60 GB state), so no flush
is needed between iterations.

roofline: the DMMA GEMM kernel (the dominant kernel, ~90 % of the flops):
achieved = sum 2MNK / sum of CUDA-event-timed GEMM launches over a profiled
pass with the streams serialised (each event bracket = one launch); at
n >= 20000 the pass covers the first --profile-steps steps (the largest
trailing matrices).  traffic = dram bytes per GEMM launch from the committed
ncu --set full capture of this config (profiles/gemm_traffic_c<cfg>.json), or
null when none exists.

cpu_baseline and --impl reference: the UNMODIFIED reference (oracle/_ref,
compiled from /root/reference/proj/src) on the box's host cores, on a bounded
sample of the same config family (same b, q and matrix kind): the faster of its
multi-threaded algorithm-by-blocks driver (randutv_ab, every host thread; needs
b | n) and its single-threaded blocked randutv().  The
config's wall time is extrapolated as F(n, b, q) / (measured GFLOP/s) and
labelled so.

--gpus N > 1 (torchrun): the 2D block-cyclic sharded factorization of ONE
matrix (strong scaling, dist.py over NCCL); --replicas runs one independent
factorization per GPU instead (weak scaling).
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

SEED_A, SEED_G = 1, 2
DMMA_PEAK_TFLOPS = 37.1  # profiles/r01_dmma_peak.jsonl: mma.sync f64 burst, 148 SMs, 1.965 GHz
METRIC = "randUTV FP64 effective GFLOP/s & time at 1/2/4/8 B200; % of FP64 TC peak"
DEFAULT_CONFIG = 5


# The contract is ONE JSON line on stdout.  Native libraries (NCCL prints its version banner
# with NCCL_DEBUG=VERSION/INFO) write to file descriptor 1 directly, so main() points fd 1 at
# stderr for the whole run and emit() writes the result line to the saved stdout.
_REAL_STDOUT = None


def capture_stdout():
    global _REAL_STDOUT
    if _REAL_STDOUT is None:
        sys.stdout.flush()
        _REAL_STDOUT = os.dup(1)
        os.dup2(2, 1)


def emit(line: dict) -> None:
    data = (json.dumps(line) + "\n").encode()
    if _REAL_STDOUT is None:
        sys.stdout.write(data.decode())
        sys.stdout.flush()
    else:
        sys.stdout.flush()
        os.write(_REAL_STDOUT, data)


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


def workload_name(n, b, q, kind, cfg):
    return f"config{cfg}: n={n} {KIND_TEXT[kind]}, b={b}, q={q}, full U/T/V"


def cliff_sigma(n):
    import numpy as np
    i = np.arange(1, n + 1)
    return np.where(i <= 3000, 1.0, 1e-3 * 0.999 ** (i - 3000.0))


def make_matrix(rutv, a, kind, seed):
    """A on the device with the reference's generators (metrics.cpp:90-110)."""
    n = a.shape[0]
    if kind == "gaussian":
        rutv.gaussian_matrix_device(a, seed)
    elif kind == "geometric":
        rutv.spectrum_matrix_device(a, seed, beta=10 ** (-12 / (n - 1)))
    else:
        rutv.spectrum_matrix_device(a, seed, sigma=cliff_sigma(n))


def config_dict(args, parallelism):
    """The `config` object of BOTH arms (identical, so the driver sees the same workload)."""
    n, b, q = args.n, args.b, args.q
    return {"workload": workload_name(n, b, q, args.kind, args.config), "n": n, "b": b, "q": q,
            "flops_per_step": args.flops, "parallelism": parallelism,
            "l2": f"inputs (A {8 * n * n / 1e9:.3g} GB + {24 * n * n / 1e9:.3g} GB state) exceed the 126 MB L2; "
                  "no flush"}


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
def sample_matrix(kind, n):
    """Bounded-sample input of the same family, generated by the C restatement
    (bit-identical to the reference's generators, tests/test_oracle_pin.py)."""
    import oracle
    if kind == "gaussian":
        return oracle.gaussian_matrix(n, n, SEED_A)
    if kind == "geometric":
        return oracle.geometric_matrix(n, n, 10 ** (-12 / (n - 1)), SEED_A)
    return oracle.spectrum_matrix(n, n, cliff_sigma(n), SEED_A)


def sample_sizes(b):
    """(n for the blocked driver, n for the AB driver) -- a few seconds of CPU work each:
    two full steps plus the ragged tail for the blocked driver, b | n for the AB driver."""
    return max(2 * b, 1000), max(4 * b, 2048)


class ReferenceSampler:
    """Times the UNMODIFIED reference on the sample; picks the faster driver once."""

    def __init__(self, b, q, kind):
        import oracle
        self.oracle, self.b, self.q, self.kind = oracle, b, q, kind
        self.n_blk, self.n_ab = sample_sizes(b)
        self.a_blk = sample_matrix(kind, self.n_blk)
        self.a_ab = sample_matrix(kind, self.n_ab)
        self.workers = os.cpu_count() or 1
        self.driver = None

    def blocked(self):
        t0 = time.perf_counter()
        self.oracle.randutv(self.a_blk, b=self.b, q=self.q, seed=SEED_G, impl="ref")
        dt = time.perf_counter() - t0
        return self.oracle.flops(self.n_blk, self.b, self.q) / dt / 1e9, dt

    def ab(self):
        t0 = time.perf_counter()
        self.oracle.ref_randutv_ab(self.a_ab, b=self.b, q=self.q, seed=SEED_G, workers=self.workers)
        dt = time.perf_counter() - t0
        return self.oracle.flops(self.n_ab, self.b, self.q) / dt / 1e9, dt

    def pick(self):
        v1, dt1 = self.blocked()
        try:
            v2, dt2 = self.ab()
        except Exception:  # the AB driver is an extra; the blocked one always exists
            v2, dt2 = -1.0, 0.0
        self.driver = "ab" if v2 > v1 else "blocked"
        self.first = (v1, dt1, v2, dt2)
        return (v2, dt2) if self.driver == "ab" else (v1, dt1)

    def sample(self):
        return self.ab() if self.driver == "ab" else self.blocked()

    def describe(self, dt):
        v1, dt1, v2, dt2 = self.first
        fam = f"b={self.b}, q={self.q}, {KIND_TEXT[self.kind]}"
        if self.driver == "ab":
            return (f"reference randutv_ab (algorithm-by-blocks, {self.workers} threads) on n={self.n_ab} of the "
                    f"config family ({fam}), {dt:.2f} s; single-thread blocked randutv() on n={self.n_blk}: "
                    f"{v1:.2f} GFLOP/s")
        return (f"reference randutv() (blocked, single thread by contract) on n={self.n_blk} of the config family "
                f"({fam}), {dt:.2f} s; randutv_ab on n={self.n_ab}: {v2:.2f} GFLOP/s")

    @property
    def cores(self):
        return self.workers if self.driver == "ab" else 1


def run_reference(args):
    """--impl reference: the reference's own CPU path on the box's host cores, on the
    same config (family sample, extrapolated to the config by the flop model)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle
    kind = "reference" if oracle.available("ref") else "port"
    vals, times = [], []
    if kind == "reference":
        rs = ReferenceSampler(args.b, args.q, args.kind)
        for i in range(args.warmup + args.steps):
            v, dt = rs.pick() if i == 0 else rs.sample()
            if i >= args.warmup:
                vals.append(v)
                times.append(dt)
        cores, sample = rs.cores, rs.describe(statistics.median(times))
    else:  # the C restatement, only if the reference library is missing
        n = sample_sizes(args.b)[0]
        a = sample_matrix(args.kind, n)
        for i in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            oracle.randutv(a, b=args.b, q=args.q, seed=SEED_G)
            dt = time.perf_counter() - t0
            if i >= args.warmup:
                vals.append(oracle.flops(n, args.b, args.q) / dt / 1e9)
                times.append(dt)
        cores, sample = os.cpu_count() or 1, f"C restatement of randutv() on n={n}"
    value = statistics.median(vals)
    cfg_s = args.flops / (value * 1e9)
    sample += (f"; value = F(sample)/t, median over the {args.steps} timed steps; config wall time extrapolated "
               f"as F(n={args.n},b={args.b},q={args.q}) / value = {cfg_s:.0f} s")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "GFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1000 * cfg_s, 1), "higher_is_better": True,
        "scaling": "strong" if args.gpus > 1 and not args.replicas else "weak", "vs_baseline": None,
        "dtype": "f64", "data": f"synthetic ({KIND_TEXT[args.kind]}, seed {SEED_A}; bounded sample of the config)",
        "config": config_dict(args, parallelism(args, args.gpus)),
        "extrapolated": {"sample_seconds_median": round(statistics.median(times), 3),
                         "config_seconds": round(cfg_s, 1), "model": "F(n,b,q) / sample GFLOP/s"},
        "cpu_baseline": {"value": round(value, 4), "unit": "GFLOP/s", "cores": cores, "kind": kind,
                         "sample": sample},
        "e2e": {"value": round(value, 4), "unit": "GFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    emit(line)
    return 0


def parallelism(args, world):
    if world <= 1:
        return "single"
    if args.replicas:
        return f"replicas x{world}"
    from paper_2104_05782_b200.dist import grid_shape
    P, Q = grid_shape(world)
    return f"2d-block-cyclic {P}x{Q}"


# ------------------------------------------------------------------- B200 --
def cm(torch, m, n, dev):
    return torch.empty((n, m), dtype=torch.float64, device=dev).T


def traffic_for(cfg):
    """dram bytes per GEMM launch from this config's committed ncu --set full capture."""
    path = os.path.join(ROOT, "profiles", f"gemm_traffic_c{cfg}.json")
    try:
        d = json.load(open(path))
        return d.get("bytes_per_launch"), os.path.relpath(path, ROOT)
    except (OSError, ValueError):
        return None, None


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", type=int, default=DEFAULT_CONFIG, choices=sorted(CONFIGS),
                    help="BASELINE.json config (default 5, the north-star single-GPU configuration)")
    ap.add_argument("--n", type=int, default=None)
    ap.add_argument("--b", type=int, default=None)
    ap.add_argument("--q", type=int, default=None)
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: one independent factorization per GPU (weak scaling) instead of the sharded "
                         "2D block-cyclic factorization of one matrix")
    ap.add_argument("--sharded", action="store_true",
                    help="the sharded driver even at N = 1 (a 1 x 1 NCCL grid; default for N > 1)")
    ap.add_argument("--e2e-steps", type=int, default=None,
                    help="timed host-pointer steps (default: K, or 2 when n >= 20000)")
    ap.add_argument("--profile-steps", type=int, default=None,
                    help="steps of the serialised GEMM-profile pass (default: all, or 12 when n >= 20000)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    capture_stdout()
    args.warmup = max(args.warmup, 0)
    cfgd = CONFIGS[args.config]
    args.n = cfgd["n"] if args.n is None else args.n
    args.b = cfgd["b"] if args.b is None else args.b
    args.q = cfgd["q"] if args.q is None else args.q
    args.kind = cfgd["kind"]
    big = args.n >= 20000
    if args.e2e_steps is None:
        args.e2e_steps = min(args.steps, 2) if big else args.steps
    if args.profile_steps is None:
        args.profile_steps = 12 if big else -1
    args.flops = flops(args.n, args.b, args.q)
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
    if (world > 1 and not args.replicas) or args.sharded:
        return run_sharded(args, torch, dist, rutv, world, rank, local, dev, args.flops)
    n, b, q, F = args.n, args.b, args.q, args.flops
    assert abs(F - rutv.flops(n, b, q)) <= 1e-9 * F

    a = cm(torch, n, n, dev)
    make_matrix(rutv, a, args.kind, SEED_A + rank)
    # T and V stacked in one buffer (V rows on top): the library factors in place
    vt = cm(torch, 2 * n, n, dev)
    t, v = vt[n:, :], vt[:n, :]
    u = cm(torch, n, n, dev)
    stream = torch.cuda.current_stream(dev)
    sh = stream.cuda_stream

    def step(max_steps=-1):
        rutv.factorize_device(a, t, u, v, b=b, q=q, seed=SEED_G, stream=sh, max_steps=max_steps)

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
    diag0 = torch.diagonal(t)[:8].cpu()

    # ---- roofline of the dominant kernel (DMMA GEMM), separate profiled pass.
    # Streams serialised (RUTV_OVERLAP=0) so each GEMM's event bracket is its own
    # launch; bounded to the first profile_steps steps at large n.
    os.environ["RUTV_GEMM_PROFILE"] = "1"
    os.environ["RUTV_OVERLAP"] = "0"
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    step(args.profile_steps)
    p1.record(stream)
    torch.cuda.synchronize()
    pass_ms = p0.elapsed_time(p1)
    os.environ["RUTV_GEMM_PROFILE"] = "0"
    os.environ["RUTV_OVERLAP"] = "1"
    gp = rutv.gemm_profile()
    gemm_tflops = gp["flops"] / (gp["ms"] / 1e3) / 1e12 if gp["ms"] > 0 else None
    traffic, tsrc = traffic_for(args.config) if (n, b, q) == tuple(CONFIGS[args.config][k] for k in "nbq") \
        else (None, None)
    roofline = {"bound": "tensor", "achieved": round(gemm_tflops, 3) if gemm_tflops else None,
                "peak": DMMA_PEAK_TFLOPS, "unit": "TFLOP/s",
                "frac": round(gemm_tflops / DMMA_PEAK_TFLOPS, 4) if gemm_tflops else None,
                "traffic": traffic, "traffic_source": tsrc, "kernel": "dgemm_kernel (+split-K reduce)",
                "gemm_ms_profiled": round(gp["ms"], 3), "gemm_launches_profiled": gp["launches"],
                "profiled_steps": args.profile_steps if args.profile_steps >= 0 else "all",
                "gemm_share_of_serialized_pass": round(gp["ms"] / pass_ms, 4) if pass_ms > 0 else None,
                "serialized_pass_ms": round(pass_ms, 3),
                "step_frac_of_peak": round(F / (ms_max / 1e3) / 1e12 / DMMA_PEAK_TFLOPS, 4),
                "peak_source": "measured DMMA burst (profiles/r01_dmma_peak.jsonl); "
                               "MEASURED_PEAKS.json has no FP64 entry"}

    # ---- e2e through the C ABI with pinned host buffers (the device tensors are
    # released first: the host-pointer call allocates its own 3 n^2 device state)
    e2e = None
    if not args.no_e2e:
        import ctypes as C
        import numpy as np
        ha = rutv.PinnedMatrix(n, n)
        torch.from_numpy(ha.array).copy_(a)  # column-major bytes of A, D2H straight into pinned memory
        del a, vt, t, v, u
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        hout = [rutv.PinnedMatrix(n, n) for _ in range(3)]
        # keep_workspace: a caller factoring repeatedly keeps the 3 n^2 device state cached
        # between calls (rutv_opts.keep_workspace) instead of re-mapping it every call
        o = rutv.make_opts(b=b, q=q, seed=SEED_G, device=local, stream=sh, keep_workspace=True)
        st = rutv.Status()
        L = rutv.lib()

        def e2e_step():
            L.rutv_b200_factorize(C.byref(o), ha.ptr, n, n, n, None, 0, hout[0].ptr, n, hout[1].ptr, n,
                                  hout[2].ptr, n, C.byref(st))
            rutv._raise(st)

        # one untimed call: maps the host path's 3 n^2 device state into the library pool
        # (kept across calls by keep_workspace); the kernels are already warm
        e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(args.e2e_steps):
            e2e_step()
        f1.record(stream)
        torch.cuda.synchronize()
        ems = torch.tensor([f0.elapsed_time(f1) / args.e2e_steps], device=dev)
        if world > 1:
            dist.all_reduce(ems, op=dist.ReduceOp.MAX)
        e2e = {"value": round(world * F / (float(ems.item()) / 1e3) / 1e9, 3), "unit": "GFLOP/s",
               "ms_per_step": round(float(ems.item()), 3), "steps": args.e2e_steps,
               "api": "rutv_b200_factorize (host pointers, pinned), keep_workspace=1",
               "h2d_bytes_per_step": 8 * n * n, "d2h_bytes_per_step": 3 * 8 * n * n}
        # sanity: the host result is the device one (same stream of deviates, deterministic)
        assert np.allclose(np.diag(hout[0].array)[:8], diag0.numpy(), rtol=1e-12, atol=0), "e2e != device run"
        for h in [ha, *hout]:
            h.close()
        rutv.release_workspace(local)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            import oracle
            if oracle.available("ref"):
                rs = ReferenceSampler(b, q, args.kind)
                v_ref, dt = rs.pick()
                cpu = {"value": round(v_ref, 4), "unit": "GFLOP/s", "cores": rs.cores, "kind": "reference",
                       "sample": rs.describe(dt) + f"; config wall time extrapolated as F/value = "
                                                   f"{F / (v_ref * 1e9):.0f} s"}
        except Exception as exc:  # the baseline is reported, never required
            cpu = {"value": None, "unit": "GFLOP/s", "cores": 1, "kind": "reference",
                   "sample": f"unavailable: {exc}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_max, 3),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": f"synthetic (device-generated {KIND_TEXT[args.kind]}, seed {SEED_A})",
            "config": config_dict(args, parallelism(args, world)),
            "e2e": e2e, "gpu_launches": launches, "clocks": clocks, "roofline": roofline,
            "cpu_baseline": cpu,
        }
        emit(line)
    if world > 1:
        dist.destroy_process_group()
    return 0


def flops(n, b, q):
    """F(n, b, q) of SURVEY.md section 8(a) (== rutv_b200_flops == oracle.flops)."""
    f, i = 0.0, 0
    while True:
        r0, s = float(i * b), float(n - i * b)
        bb, nn = float(b), float(n)
        if s <= 0:
            break
        if s <= bb:
            f += 2 * r0 * s * s + 4 * nn * s * s
            break
        f += 2 * s * s * bb * (1 + 2 * q)
        f += 4 * s * s * bb + 2 * s * bb * bb
        f += 4 * r0 * s * bb + 2 * r0 * bb * bb
        f += 4 * nn * s * bb + 2 * nn * bb * bb
        f += 4 * s * bb * (s - bb) + 2 * bb * bb * (s - bb)
        f += 4 * nn * s * bb + 2 * nn * bb * bb
        f += 2 * bb * bb * (s - bb) + 2 * r0 * bb * bb + 4 * nn * bb * bb
        f += 4 * bb * bb * (s - bb / 3)
        i += 1
    return f


# ---------------------------------------------------------- sharded (2D) --
def run_sharded(args, torch, dist, rutv, world, rank, local, dev, F):
    """ONE matrix on the P x Q block-cyclic grid: the C++ sharded driver (dist.cu,
    rutv_b200_factorize_dist) over NCCL, one rank per GPU -- strong scaling.
    value = F / (max over ranks of the device time of one factorization)."""
    from paper_2104_05782_b200.dist import grid_shape
    n, b, q = args.n, args.b, args.q
    P, Q = grid_shape(world)
    uid = [rutv.nccl_unique_id() if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(uid, src=0)
    ctx = rutv.DistContext(uid[0], P, Q, rank, local)
    log(f"[bench] rank {rank}: NCCL grid {P}x{Q} communicators up on cuda:{local}")
    mr, mc = rutv.grid_local_shape(n, b, P, Q, rank)
    full = cm(torch, n, n, dev)
    make_matrix(rutv, full, args.kind, SEED_A)  # same matrix on every rank (deterministic generator)
    a_loc = cm(torch, mr, mc, dev)
    rutv.grid_copy(full, a_loc, n, b, P, Q, rank, to_local=True)
    del full
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    vt = cm(torch, 2 * mr, mc, dev)  # [V; T] stacked: factored in place
    t_loc, v_loc = vt[mr:, :], vt[:mr, :]
    u_loc = cm(torch, mr, mc, dev)
    stream = torch.cuda.current_stream(dev)
    sh = stream.cuda_stream

    def step(a_src=None):
        ctx.factorize(n, a_loc if a_src is None else a_src, t_loc, u_loc, v_loc, b=b, q=q, seed=SEED_G, stream=sh)

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
    ms_t = torch.tensor([e0.elapsed_time(e1) / args.steps], device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms = float(ms_t.item())
    # e2e: this rank's blocks from pinned host memory, its T, U, V blocks back to pinned host memory
    e2e = None
    if not args.no_e2e:
        ha = rutv.PinnedMatrix(mr, mc)
        rutv.copy_matrix_async(ha.array, a_loc, sh)
        hout = [rutv.PinnedMatrix(mr, mc) for _ in range(3)]
        dbuf = cm(torch, mr, mc, dev)
        steps_e = args.e2e_steps
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        for _ in range(steps_e):
            rutv.copy_matrix_async(dbuf, ha.array, sh)  # pinned host -> HBM on the timed stream
            step(dbuf)
            for h, d in zip(hout, (t_loc, u_loc, v_loc)):
                rutv.copy_matrix_async(h.array, d, sh)
        f1.record(stream)
        torch.cuda.synchronize()
        ems = torch.tensor([f0.elapsed_time(f1) / steps_e], device=dev)
        if world > 1:
            dist.all_reduce(ems, op=dist.ReduceOp.MAX)
        e2e = {"value": round(F / (float(ems.item()) / 1e3) / 1e9, 3), "unit": "GFLOP/s",
               "ms_per_step": round(float(ems.item()), 3), "steps": steps_e,
               "h2d_bytes_per_step": 8 * mr * mc, "d2h_bytes_per_step": 3 * 8 * mr * mc, "per_rank": True}
        for h in [ha, *hout]:
            h.close()
    ctx.close()
    if rank == 0:
        value = F / (ms / 1e3) / 1e9
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": "GFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": f"synthetic (device-generated {KIND_TEXT[args.kind]}, seed {SEED_A})",
            "config": config_dict(args, f"2d-block-cyclic {P}x{Q}"),
            "e2e": e2e, "gpu_launches": launches, "clocks": clk.summary(),
            "roofline": {"bound": "tensor", "achieved": round(value / 1e3 / world, 3), "peak": DMMA_PEAK_TFLOPS,
                         "unit": "TFLOP/s", "frac": round(value / 1e3 / world / DMMA_PEAK_TFLOPS, 4),
                         "traffic": None, "kernel": "whole sharded factorization per GPU (dist.cu)",
                         "step_frac_of_peak": round(value / 1e3 / world / DMMA_PEAK_TFLOPS, 4)},
            "cpu_baseline": None,
        }
        emit(line)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
