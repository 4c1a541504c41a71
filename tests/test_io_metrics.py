"""The data format and quality metrics either side of the path.

* .rutv (proj/src/matrix_io.cpp:40-70): the oracle restatement and the
  library's native reader/writer (host mode, no GPU needed) against files the
  UNMODIFIED reference wrote (tests/golden/*.rutv, tests/golden/make_golden.py),
  byte for byte, plus the reference's IoError cases (bad magic, truncated
  header / payload, implausible dimensions, trailing bytes) -> OSError.
* lowrank_error (proj/src/metrics.cpp:32-46): the oracle restatement against the
  reference's values (tests/golden/lowrank_r64.npz); the device version in the
  -m gpu tests below.
"""
import os

import numpy as np
import pytest

import oracle
import paper_2104_05782_b200 as rutv

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _gold(name):
    return os.path.join(GOLD, name)


def test_oracle_rutv_matches_reference_files():
    a = oracle.gaussian_matrix(5, 3, 77)
    raw = open(_gold("g5x3.rutv"), "rb").read()
    assert oracle.rutv_bytes(a) == raw
    assert np.array_equal(oracle.parse_rutv(raw), a)
    raw0 = open(_gold("empty0x4.rutv"), "rb").read()
    assert oracle.rutv_bytes(np.zeros((0, 4))) == raw0 and len(raw0) == 20
    assert oracle.parse_rutv(raw0).shape == (0, 4)


def test_native_reader_host_mode_bit_exact():
    a = rutv.read_rutv(_gold("g5x3.rutv"))
    assert a.shape == (5, 3) and np.array_equal(a, oracle.gaussian_matrix(5, 3, 77))
    assert rutv.read_rutv(_gold("empty0x4.rutv")).shape == (0, 4)


def test_native_writer_host_mode_bit_exact(tmp_path):
    for shape, seed in [((5, 3), 77), ((1, 1), 3), ((13, 7), 5)]:
        a = oracle.gaussian_matrix(*shape, seed)
        p = str(tmp_path / f"x{shape[0]}_{shape[1]}.rutv")
        rutv.write_rutv(p, a)
        assert open(p, "rb").read() == oracle.rutv_bytes(a)
        if oracle.available("ref"):
            assert np.array_equal(oracle.ref_read_rutv(p), a)
    # a strided (non-contiguous) view is written column-major like the reference's view
    big = oracle.gaussian_matrix(9, 9, 1)
    p = str(tmp_path / "view.rutv")
    rutv.write_rutv(p, big[2:7, 1:5])
    assert open(p, "rb").read() == oracle.rutv_bytes(big[2:7, 1:5])
    p0 = str(tmp_path / "e.rutv")
    rutv.write_rutv(p0, np.zeros((0, 4)))
    assert open(p0, "rb").read() == open(_gold("empty0x4.rutv"), "rb").read()


@pytest.mark.parametrize("payload,msg", [
    (b"RUTX" + b"\0" * 16, "bad magic"),
    (b"RU", "bad magic"),
    (b"RUTV" + b"\1\0\0\0", "truncated header"),
    (b"RUTV" + np.array([2, 2], "<u8").tobytes() + b"\0" * 24, "truncated header"),
    (b"RUTV" + np.array([1 << 31, 1], "<u8").tobytes(), "implausible dimensions"),
    (b"RUTV" + np.array([1, 1], "<u8").tobytes() + b"\0" * 9, "trailing bytes"),
])
def test_reader_errors_are_ioerror(tmp_path, payload, msg):
    p = str(tmp_path / "bad.rutv")
    open(p, "wb").write(payload)
    with pytest.raises(OSError, match=msg):
        rutv.read_rutv(p)
    with pytest.raises(OSError, match=msg):
        oracle.parse_rutv(payload)
    if oracle.available("ref"):
        with pytest.raises(oracle.OracleError):
            oracle.ref_read_rutv(p)


def test_missing_file_is_ioerror(tmp_path):
    with pytest.raises(OSError, match="cannot open"):
        rutv.read_rutv(str(tmp_path / "nope.rutv"))
    with pytest.raises(OSError, match="for writing"):
        rutv.write_rutv(str(tmp_path / "no_dir" / "x.rutv"), np.eye(2))


def test_oracle_lowrank_error_matches_reference_values():
    r = np.load(_gold("randutv_r64_b16_q2.npz"))
    g = np.load(_gold("lowrank_r64.npz"))
    nf = np.linalg.norm(r["a"])
    for k, fro, spec in zip(g["ks"], g["fro"], g["spec"]):
        assert abs(oracle.lowrank_error(r["a"], r["t"], r["u"], r["v"], int(k)) - fro) <= 1e-13 * nf
        assert abs(oracle.lowrank_error(r["a"], r["t"], r["u"], r["v"], int(k), "spec") - spec) <= 1e-12 * nf
    with pytest.raises(IndexError):
        oracle.lowrank_error(r["a"], r["t"], r["u"], r["v"], 65)


def test_optimal_error_and_csv():
    sig = np.array([4.0, 3.0, 2.0, 1.0])
    assert rutv.optimal_error(sig, 1) == oracle.optimal_error(sig, 1) == np.sqrt(14.0)
    assert rutv.optimal_error(sig, 2, "spectral") == 2.0 and rutv.optimal_error(sig, 4) == 0.0
    rows = [{"k": 1, "err_utv": 1.5, "err_opt": 1.0, "ratio": 1.5, "diag_relerr": 0.0}]
    assert rutv.to_csv(rows) == "k,err_utv,err_opt,ratio,diag_relerr\n1,1.5,1,1.5,0\n"


# ------------------------------------------------------------------------ GPU
@pytest.mark.gpu
def test_device_rutv_roundtrip_multi_chunk(tmp_path):
    import torch
    n = 3000  # 72 MB: two 64 MB staging chunks
    a = torch.empty((n, n), dtype=torch.float64, device="cuda").T
    rutv.gaussian_matrix_device(a, 9)
    p = str(tmp_path / "big.rutv")
    rutv.write_rutv(p, a)
    assert os.path.getsize(p) == 20 + 8 * n * n
    host = rutv.read_rutv(p)
    assert np.array_equal(host, a.cpu().numpy())
    b = rutv.read_rutv(p, device="cuda")
    assert b.stride(0) == 1 and torch.equal(a, b)
    # the file is exactly what the restated format gives for the same bits
    sub = host[:7, :5]
    p2 = str(tmp_path / "sub.rutv")
    rutv.write_rutv(p2, a[:7, :5])
    assert open(p2, "rb").read() == oracle.rutv_bytes(sub)


@pytest.mark.gpu
def test_device_lowrank_error_matches_reference_values():
    import torch
    r = np.load(_gold("randutv_r64_b16_q2.npz"))
    g = np.load(_gold("lowrank_r64.npz"))
    dev = {k: torch.from_numpy(np.asfortranarray(r[k]).T.copy()).cuda().T for k in "atuv"}
    nf = np.linalg.norm(r["a"])
    for k, fro, spec in zip(g["ks"], g["fro"], g["spec"]):
        e = rutv.lowrank_error(dev["a"], dev["t"], dev["u"], dev["v"], int(k))
        assert abs(e - fro) <= 1e-13 * nf, (k, e, fro)
        e = rutv.lowrank_error(dev["a"], dev["t"], dev["u"], dev["v"], int(k), "spectral")
        assert abs(e - spec) <= 1e-12 * nf, (k, e, spec)
    with pytest.raises(IndexError):
        rutv.lowrank_error(dev["a"], dev["t"], dev["u"], dev["v"], 65)


@pytest.mark.gpu
def test_quality_report_on_known_spectrum():
    import torch
    n, b, q, beta = 600, 64, 2, 0.97
    a = torch.empty((n, n), dtype=torch.float64, device="cuda").T
    rutv.spectrum_matrix_device(a, 5, beta=beta)
    t, u, v = (torch.empty((n, n), dtype=torch.float64, device="cuda").T for _ in range(3))
    rutv.factorize_device(a, t, u, v, b=b, q=q, seed=3)
    sig = beta ** np.arange(n)
    rows = rutv.quality_report(a, t, u, v, [1, 10, 64, 200], sig)
    host = {k: x.cpu().numpy() for k, x in zip("atuv", (a, t, u, v))}
    for r in rows:
        want = oracle.lowrank_error(host["a"], host["t"], host["u"], host["v"], r["k"])
        assert abs(r["err_utv"] - want) <= 1e-12 * np.sqrt(np.sum(sig ** 2))
        assert r["err_opt"] == pytest.approx(oracle.optimal_error(sig, r["k"]), rel=1e-14)
        assert 1.0 - 1e-9 <= r["ratio"] < 1.5      # randUTV with q=2 is near-optimal here
    csv = rutv.to_csv(rows)
    assert csv.startswith("k,err_utv,err_opt,ratio,diag_relerr\n") and csv.count("\n") == 5
