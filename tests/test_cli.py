"""The CLI mirror (python -m paper_2104_05782_b200): bench CSV format of
proj/src/bench.cpp:69-93 and the factorize round trip of randutv_cli.cpp:89-114."""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
from paper_2104_05782_b200 import __main__ as cli

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_csv_format_and_median_flag():
    rows = [{"algo": "b200", "n": 100, "b": 32, "q": 1, "workers": 1, "build_uv": True, "seconds": s,
             "scaled": cli.scaled_time(s, 100), "median": False, "gflops": 1.5} for s in (0.3, 0.1, 0.2)]
    cli.flag_medians(rows, 0)
    assert [r["median"] for r in rows] == [False, False, True]   # sorted 0.1, 0.2, 0.3 -> index 1
    rows2 = [dict(rows[0], seconds=0.4, median=False), dict(rows[0], seconds=0.5, median=False)]
    cli.flag_medians(rows2, 0)                                    # R = 2 -> index (2-1)//2 = 0
    assert [r["median"] for r in rows2] == [True, False]
    csv = cli.bench_csv(rows)
    lines = csv.splitlines()
    assert lines[0] == "algo,n,b,q,workers,build_uv,seconds,scaled,median,gflops"
    assert lines[1].split(",")[:6] == ["b200", "100", "32", "1", "1", "1"]
    assert float(lines[1].split(",")[6]) == 0.3 and lines[3].split(",")[8] == "1"
    assert cli.scaled_time(2.0, 100) == 2.0 / 1e6 * 1e10


def test_usage_errors_exit_2():
    assert cli.main(["bench"]) == 2               # --sizes is required
    assert cli.main(["nosuchcommand"]) == 2


@pytest.mark.gpu
def test_cli_bench_and_factorize_on_gpu(tmp_path):
    env = dict(os.environ, PYTHONPATH=ROOT)
    out = subprocess.run([sys.executable, "-m", "paper_2104_05782_b200", "bench", "--sizes", "200,256",
                          "--b", "32,64", "--q", "1", "--repeats", "3"], capture_output=True, text=True,
                         env=env, cwd=ROOT, timeout=300)
    assert out.returncode == 0, out.stderr
    lines = out.stdout.strip().splitlines()
    assert lines[0].startswith("algo,n,b,q,workers,build_uv,seconds,scaled,median")
    assert len(lines) == 1 + 2 * 2 * 3
    assert sum(int(l.split(",")[8]) for l in lines[1:]) == 4   # one median per configuration
    a = oracle.gaussian_matrix(120, 120, 3)
    p = str(tmp_path / "a.rutv")
    open(p, "wb").write(oracle.rutv_bytes(a))
    pre = str(tmp_path / "res")
    out = subprocess.run([sys.executable, "-m", "paper_2104_05782_b200", "factorize", p, "--out", pre,
                          "--b", "32", "--q", "2", "--seed", "5"], capture_output=True, text=True, env=env,
                         cwd=ROOT, timeout=300)
    assert out.returncode == 0, out.stderr
    assert out.stdout.startswith("factored 120 x 120 (b200, b=32, q=2)")
    t, u, v = (oracle.parse_rutv(open(f"{pre}_{x}.rutv", "rb").read()) for x in "TUV")
    assert np.linalg.norm(a - u @ t @ v.T) / np.linalg.norm(a) < 1e-13
    tr, _, _ = oracle.randutv(a, b=32, q=2, seed=5)
    assert np.max(np.abs(np.abs(np.diag(t)) - np.abs(np.diag(tr))) / np.abs(np.diag(tr))) < 1e-9
    bad = subprocess.run([sys.executable, "-m", "paper_2104_05782_b200", "factorize", str(tmp_path / "none.rutv")],
                         capture_output=True, text=True, env=env, cwd=ROOT, timeout=300)
    assert bad.returncode == 2 and "cannot open" in bad.stderr
