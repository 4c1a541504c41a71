"""Command line mirror of the reference CLI's hot-path subcommands on the B200.

    python -m paper_2104_05782_b200 factorize A.rutv [--out utv] [--b 128] [--q 1] [--seed 0] [--no-uv]
    python -m paper_2104_05782_b200 bench --sizes 2000,4000 [--b 128] [--q 1] [--repeats 3] [--seed 0]
                                          [--no-uv] [--csv out.csv]

``factorize`` follows proj/tools/randutv_cli.cpp:89-114 (read the matrix, factor,
write <out>_{T,U,V}.rutv, print one summary line).  ``bench`` follows
run_bench / bench_csv (proj/src/bench.cpp:32-93): one Gaussian matrix per size
from ``--seed`` (metrics.cpp:90-93), every (n, b, q) timed ``--repeats`` times
around the call (the reference times with steady_clock around randutv(); here
the device call including its final synchronisation), the median-seconds
repeat flagged, CSV header ``algo,n,b,q,workers,build_uv,seconds,scaled,median``
plus a trailing ``gflops`` column (F(n, b, q) / seconds; the flop
model counts U and V, so it is left empty for --no-uv rows).  ``algo`` is
``b200``; ``workers`` is 1 (one GPU).  Exit codes as the reference: 0 success,
2 usage or I/O error.
"""
from __future__ import annotations

import argparse
import os
import sys
import time


def scaled_time(seconds: float, n: int) -> float:
    """metrics.cpp:145-149: seconds / n^3 * 1e10."""
    if n < 1:
        raise ValueError("scaled_time: n must be >= 1")
    return seconds / (float(n) ** 3) * 1e10


def bench_csv(rows: list[dict]) -> str:
    """bench.cpp:83-93 format (%.17g seconds / scaled) + gflops."""
    out = ["algo,n,b,q,workers,build_uv,seconds,scaled,median,gflops"]
    for r in rows:
        gf = "" if r.get("gflops") is None else "%.6g" % r["gflops"]
        out.append("%s,%d,%d,%d,%d,%d,%.17g,%.17g,%d,%s" % (
            r["algo"], r["n"], r["b"], r["q"], r["workers"], 1 if r["build_uv"] else 0, r["seconds"],
            r["scaled"], 1 if r["median"] else 0, gf))
    return "\n".join(out) + "\n"


def flag_medians(rows: list[dict], first: int) -> None:
    """bench.cpp:69-75: the repeat at index (R - 1) / 2 of the seconds-sorted order is the median."""
    idx = sorted(range(first, len(rows)), key=lambda i: rows[i]["seconds"])
    rows[idx[(len(idx) - 1) // 2]]["median"] = True


def _int_list(s: str) -> list[int]:
    return [int(x) for x in s.split(",") if x.strip()]


def cmd_factorize(a) -> int:
    import torch
    import paper_2104_05782_b200 as rutv
    x = rutv.read_rutv(a.input, device="cuda")
    m, n = x.shape
    b = a.b if a.b > 0 else 128
    t = torch.empty((n, m), dtype=torch.float64, device="cuda").T
    u = None if a.no_uv else torch.empty((m, m), dtype=torch.float64, device="cuda").T
    v = None if a.no_uv else torch.empty((n, n), dtype=torch.float64, device="cuda").T
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rutv.factorize_device(x, t, u, v, b=b, q=a.q, seed=a.seed)
    torch.cuda.synchronize()
    secs = time.perf_counter() - t0
    written = [a.out + "_T.rutv"]
    rutv.write_rutv(written[0], t)
    if not a.no_uv:
        rutv.write_rutv(a.out + "_U.rutv", u)
        rutv.write_rutv(a.out + "_V.rutv", v)
        written += [a.out + "_U.rutv", a.out + "_V.rutv"]
    print("factored %d x %d (b200, b=%d, q=%d) in %.3f s; wrote %s" % (m, n, b, a.q, secs, ", ".join(written)))
    return 0


def cmd_bench(a) -> int:
    import torch
    import paper_2104_05782_b200 as rutv
    if a.repeats < 1:
        raise ValueError("bench repeats must be positive")
    sizes, bs, qs = _int_list(a.sizes), _int_list(a.b), _int_list(a.q)
    if not sizes or not bs or not qs:
        raise ValueError("bench plan has an empty axis")
    rows: list[dict] = []
    for n in sizes:
        if n < 1:
            raise ValueError("bench size must be positive")
        x = torch.empty((n, n), dtype=torch.float64, device="cuda").T
        rutv.gaussian_matrix_device(x, a.seed)
        t = torch.empty((n, n), dtype=torch.float64, device="cuda").T
        u = None if a.no_uv else torch.empty((n, n), dtype=torch.float64, device="cuda").T
        v = None if a.no_uv else torch.empty((n, n), dtype=torch.float64, device="cuda").T
        for b in bs:
            for q in qs:
                rutv.factorize_device(x, t, u, v, b=b, q=q, seed=a.seed)  # warm-up (module load, pools)
                first = len(rows)
                for _ in range(a.repeats):
                    torch.cuda.synchronize()
                    t0 = time.perf_counter()
                    rutv.factorize_device(x, t, u, v, b=b, q=q, seed=a.seed)
                    torch.cuda.synchronize()
                    secs = time.perf_counter() - t0
                    rows.append({"algo": "b200", "n": n, "b": b, "q": q, "workers": 1, "build_uv": not a.no_uv,
                                 "seconds": secs, "scaled": scaled_time(secs, n), "median": False,
                                 "gflops": None if a.no_uv else rutv.flops(n, b, q) / secs / 1e9})
                flag_medians(rows, first)
        del x, t, u, v
    csv = bench_csv(rows)
    if not a.csv:
        sys.stdout.write(csv)
    else:
        try:
            with open(a.csv, "w", newline="") as f:
                f.write(csv)
        except OSError as exc:
            raise OSError(f"cannot open {a.csv} for writing") from exc
        print(f"wrote {len(rows)} rows to {a.csv}")
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2104_05782_b200",
                                 description="B200 randUTV: factorize .rutv files, benchmark sweeps (CSV)")
    sub = ap.add_subparsers(dest="cmd", required=True)
    f = sub.add_parser("factorize", help="factor a matrix file as A = U T V'")
    f.add_argument("input")
    f.add_argument("--out", default="utv")
    f.add_argument("--b", type=int, default=0)
    f.add_argument("--q", type=int, default=1)
    f.add_argument("--seed", type=int, default=0)
    f.add_argument("--no-uv", action="store_true")
    bch = sub.add_parser("bench", help="timed factorization sweep, CSV output")
    bch.add_argument("--sizes", required=True)
    bch.add_argument("--b", default="128")
    bch.add_argument("--q", default="1")
    bch.add_argument("--repeats", type=int, default=3)
    bch.add_argument("--seed", type=int, default=0)
    bch.add_argument("--no-uv", action="store_true")
    bch.add_argument("--csv", default="")
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:
        return 0 if e.code == 0 else 2
    try:
        return cmd_factorize(a) if a.cmd == "factorize" else cmd_bench(a)
    except (OSError, ValueError, IndexError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
