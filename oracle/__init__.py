"""CPU oracle for the blocked randUTV path -- TEST INFRASTRUCTURE ONLY.

Two checkers live here, both exposed through the same Python signatures:

* ``impl="port"``: ``rutv_oracle.c``, our plain-C restatement of the reference
  algorithm (every function cites the reference file:line it follows);
* ``impl="ref"``: ``_ref/librandutv_ref.so``, the UNMODIFIED reference sources
  from /root/reference/proj compiled by ``oracle/Makefile`` (git-ignored,
  shipped to the GPU box prebuilt).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
legs may import this module; the product package never does.  Parity is
pinned in ``tests/test_oracle_pin.py``: port == ref bit for bit, and both ==
the committed golden fixtures in ``tests/golden/``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "librutv_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "librandutv_ref.so")
REF_SRC = "/root/reference/proj"

STATUS = {0: "OK", 1: "CONFIG", 2: "SHAPE", 3: "INDEX", 4: "CONVERGENCE", 7: "OOM", 9: "INTERNAL"}


class OracleError(RuntimeError):
    def __init__(self, code: int, residual: float = 0.0):
        super().__init__(f"oracle status {STATUS.get(code, code)} (residual {residual})")
        self.code = code
        self.residual = residual


def build(ref: bool = True) -> None:
    """Compile the C port (always) and the reference (when its sources exist)."""
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True)
    if ref and os.path.isdir(REF_SRC):
        subprocess.run(["make", "-s", "-C", HERE, "ref"], check=True)


_libs: dict[str, C.CDLL] = {}
_D = C.POINTER(C.c_double)
_I64 = C.c_int64


def _lib(impl: str) -> C.CDLL:
    if impl in _libs:
        return _libs[impl]
    path = PORT_SO if impl == "port" else REF_SO
    if not os.path.exists(path):
        if impl == "port" or os.path.isdir(REF_SRC):
            build(ref=impl == "ref")
    if not os.path.exists(path):
        raise FileNotFoundError(f"oracle library {path} not built")
    lib = C.CDLL(path)
    pre = "ora_" if impl == "port" else "ref_"
    f = getattr(lib, pre + "randutv")
    if impl == "port":
        f.argtypes = [_D, _I64, _I64, _I64, _I64, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_int,
                      C.c_int, _D, _D, _D, _D]
    else:
        f.argtypes = [_D, _I64, _I64, _I64, _I64, C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_int,
                      _D, _D, _D, _D]
        lib.ref_randutv_steps.argtypes = [_D, _I64, _I64, _I64, _I64, C.c_int, C.c_int, C.c_int,
                                          C.c_uint64, C.c_int, _D, _D, _D, _D]
        lib.ref_hqr.argtypes = [_D, _I64, _I64, _I64, _D, _D, _D]
    getattr(lib, pre + "normal_fill").argtypes = [C.c_uint64, C.c_uint64, _D, _I64]
    getattr(lib, pre + "gaussian_matrix").argtypes = [_I64, _I64, C.c_uint64, _D]
    getattr(lib, pre + "geometric_matrix").argtypes = [_I64, _I64, C.c_double, C.c_uint64, _D]
    getattr(lib, pre + "svd_block").argtypes = [_D, _I64, _I64, C.c_double, C.c_int, _D, _D, _D, _D]
    getattr(lib, pre + "svd_full").argtypes = [_D, _I64, _I64, _I64, _D, _D, _D]
    getattr(lib, pre + "gemm").argtypes = [C.c_double, C.c_int, _D, _I64, _I64, _I64, C.c_int, _D,
                                           _I64, _I64, _I64, C.c_double, _D, _I64, _I64, _I64]
    if impl == "port":
        lib.ora_hqr_inplace.argtypes = [_D, _I64, _I64, _I64, _D]
        lib.ora_form_wy_t.argtypes = [_D, _I64, _I64, _D, _I64, _D]
        lib.ora_stream_length.argtypes = [_I64, _I64, _I64]
        lib.ora_stream_length.restype = _I64
        lib.ora_flops.argtypes = [_I64, _I64, C.c_int]
        lib.ora_flops.restype = C.c_double
        lib.ora_normal_at.argtypes = [C.c_uint64, C.c_uint64]
        lib.ora_normal_at.restype = C.c_double
        lib.ora_spectrum_matrix.argtypes = [_I64, _I64, C.c_double, _D, C.c_uint64, _D]
        lib.ora_apply_q_right.argtypes = [_D, _I64, _I64, _D, _I64, _D, _I64, _I64]
        lib.ora_apply_qt_left.argtypes = [_D, _I64, _I64, _D, _I64, _D, _I64, _I64]
    _libs[impl] = lib
    return lib


def _p(x: np.ndarray):
    return x.ctypes.data_as(_D)


def _f(a) -> np.ndarray:
    return np.asfortranarray(np.asarray(a, dtype=np.float64))


def available(impl: str) -> bool:
    try:
        _lib(impl)
        return True
    except (FileNotFoundError, OSError, subprocess.CalledProcessError):
        return False


def randutv(a, *, b: int = 128, q: int = 1, seed: int = 0, build_u: bool = True,
            build_v: bool = True, qr_prepass: bool = False, max_steps: int = -1,
            impl: str = "port"):
    """randutv::randutv (proj/src/randutv_blocked.cpp:84-157) -> (T, U, V).

    ``max_steps >= 0`` stops after that many loop iterations (first-k-step
    parity for sizes the full oracle cannot finish)."""
    a = _f(a)
    m, n = a.shape
    t = np.zeros((m, n), order="F")
    u = np.zeros((m, m), order="F") if build_u else np.zeros((1, 1), order="F")
    v = np.zeros((n, n), order="F") if build_v else np.zeros((1, 1), order="F")
    res = np.zeros(1)
    lib = _lib(impl)
    if impl == "port":
        rc = lib.ora_randutv(_p(a), m, n, max(m, 1), b, q, int(build_u), int(build_v), seed,
                             int(qr_prepass), max_steps, _p(t), _p(u), _p(v), _p(res))
    elif max_steps >= 0 and not qr_prepass:
        rc = lib.ref_randutv_steps(_p(a), m, n, max(m, 1), b, q, int(build_u), int(build_v),
                                   seed, max_steps, _p(t), _p(u), _p(v), _p(res))
    else:
        rc = lib.ref_randutv(_p(a), m, n, max(m, 1), b, q, int(build_u), int(build_v), seed,
                             int(qr_prepass), _p(t), _p(u), _p(v), _p(res))
    if rc != 0:
        raise OracleError(rc, float(res[0]))
    return t, (u if build_u else None), (v if build_v else None)


def normal_stream(seed: int, pos: int, count: int, impl: str = "port") -> np.ndarray:
    """Deviates pos..pos+count-1 of RngState(seed) (proj/src/rng.cpp:29-53)."""
    out = np.zeros(count)
    lib = _lib(impl)
    getattr(lib, ("ora_" if impl == "port" else "ref_") + "normal_fill")(seed, pos, _p(out), count)
    return out


def stream_length(m: int, n: int, b: int) -> int:
    """Number of G deviates the blocked driver draws for an m x n input."""
    return int(_lib("port").ora_stream_length(m, n, b))


def flops(n: int, b: int, q: int) -> float:
    """F(n, b, q): SURVEY.md section 8(a) algorithmic flop count (U and V built)."""
    return float(_lib("port").ora_flops(n, b, q))


def gaussian_matrix(m: int, n: int, seed: int, impl: str = "port") -> np.ndarray:
    """proj/src/metrics.cpp:90-93."""
    a = np.zeros((m, n), order="F")
    getattr(_lib(impl), ("ora_" if impl == "port" else "ref_") + "gaussian_matrix")(m, n, seed, _p(a))
    return a


def geometric_matrix(m: int, n: int, beta: float, seed: int, impl: str = "port") -> np.ndarray:
    """proj/src/metrics.cpp:95-110: Q1 diag(beta^i) Q2^T, Haar Q from form_q(hqr(G))."""
    a = np.zeros((m, n), order="F")
    rc = getattr(_lib(impl), ("ora_" if impl == "port" else "ref_") + "geometric_matrix")(
        m, n, beta, seed, _p(a))
    if rc != 0:
        raise OracleError(rc)
    return a


def spectrum_matrix(m: int, n: int, sigma, seed: int) -> np.ndarray:
    """geometric_matrix's construction with an explicit spectrum (config 4)."""
    a = np.zeros((m, n), order="F")
    s = np.ascontiguousarray(sigma, dtype=np.float64)
    rc = _lib("port").ora_spectrum_matrix(m, n, 0.0, _p(s), seed, _p(a))
    if rc != 0:
        raise OracleError(rc)
    return a


def svd_block(a, tol: float = 1e-15, max_sweeps: int = 30, impl: str = "port"):
    """proj/src/jacobi_svd.cpp:39-148 -> (U, sigma, V)."""
    a = _f(a)
    n = a.shape[0]
    u = np.zeros((n, n), order="F")
    v = np.zeros((n, n), order="F")
    s = np.zeros(max(n, 1))
    res = np.zeros(1)
    rc = getattr(_lib(impl), ("ora_" if impl == "port" else "ref_") + "svd_block")(
        _p(a), n, max(n, 1), tol, max_sweeps, _p(u), _p(s), _p(v), _p(res))
    if rc != 0:
        raise OracleError(rc, float(res[0]))
    return u, s[:n], v


def svd_full(a, impl: str = "port"):
    """proj/src/jacobi_svd.cpp:185-192 -> (U m x m, sigma, V n x n)."""
    a = _f(a)
    m, n = a.shape
    u = np.zeros((m, m), order="F")
    v = np.zeros((n, n), order="F")
    s = np.zeros(max(min(m, n), 1))
    rc = getattr(_lib(impl), ("ora_" if impl == "port" else "ref_") + "svd_full")(
        _p(a), m, n, max(m, 1), _p(u), _p(s), _p(v))
    if rc != 0:
        raise OracleError(rc)
    return u, s[:min(m, n)], v


def hqr(a, impl: str = "port"):
    """hqr_inplace + form_wy_t (proj/src/householder.cpp:48-97) -> (packed QR, tau, Twy)."""
    a = _f(a)
    m, n = a.shape
    p = min(m, n)
    tau = np.zeros(max(p, 1))
    twy = np.zeros((p, p), order="F")
    if impl == "port":
        qr = a.copy(order="F")
        _lib("port").ora_hqr_inplace(_p(qr), m, n, max(m, 1), _p(tau))
        _lib("port").ora_form_wy_t(_p(qr), m, max(m, 1), _p(tau), p, _p(twy))
    else:
        qr = np.zeros((m, n), order="F")
        rc = _lib("ref").ref_hqr(_p(a), m, n, max(m, 1), _p(qr), _p(tau), _p(twy))
        if rc != 0:
            raise OracleError(rc)
    return qr, tau[:p], twy


def gemm(alpha, ta, a, tb, b, beta, c, impl: str = "port") -> np.ndarray:
    """proj/src/gemm.cpp:21-75 on copies; returns the new C."""
    a, b = _f(a), _f(b)
    c = _f(c).copy(order="F")
    m, n = c.shape
    rc = getattr(_lib(impl), ("ora_" if impl == "port" else "ref_") + "gemm")(
        alpha, int(ta), _p(a), a.shape[0], a.shape[1], max(a.shape[0], 1), int(tb), _p(b),
        b.shape[0], b.shape[1], max(b.shape[0], 1), beta, _p(c), m, n, max(m, 1))
    if rc != 0:
        raise OracleError(rc)
    return c


def apply_q_right(qr, twy, b) -> np.ndarray:
    """householder.cpp:129-140: B <- B Q (returns a new array)."""
    qr, twy = _f(qr), _f(twy)
    b = _f(b).copy(order="F")
    s, p = qr.shape[0], twy.shape[0]
    _lib("port").ora_apply_q_right(_p(qr), s, max(s, 1), _p(twy), p, _p(b), b.shape[0],
                                   max(b.shape[0], 1))
    return b


def apply_qt_left(qr, twy, b) -> np.ndarray:
    """householder.cpp:103-114: B <- Q' B (returns a new array)."""
    qr, twy = _f(qr), _f(twy)
    b = _f(b).copy(order="F")
    s, p = qr.shape[0], twy.shape[0]
    _lib("port").ora_apply_qt_left(_p(qr), s, max(s, 1), _p(twy), p, _p(b), b.shape[1],
                                   max(b.shape[0], 1))
    return b


def form_wy_t(qr, tau) -> np.ndarray:
    """householder.cpp:76-97 on a packed QR: Twy (p x p)."""
    qr = _f(qr)
    tau = np.ascontiguousarray(tau, dtype=np.float64)
    p = tau.size
    twy = np.zeros((p, p), order="F")
    _lib("port").ora_form_wy_t(_p(qr), qr.shape[0], max(qr.shape[0], 1), _p(tau), p, _p(twy))
    return twy


# ------------------------------------------------------------------ data format + metrics
def rutv_bytes(a) -> bytes:
    """matrix_io.cpp:40-50 restated: b"RUTV", u64 LE rows, u64 LE cols, column-major f64 LE."""
    a = _f(a)
    m, n = a.shape
    return b"RUTV" + np.array([m, n], dtype="<u8").tobytes() + a.astype("<f8").tobytes(order="F")


def parse_rutv(data: bytes) -> np.ndarray:
    """matrix_io.cpp:52-70 restated (same checks, IoError -> OSError with the reference's text)."""
    if len(data) < 4 or data[:4] != b"RUTV":
        raise OSError("bad magic")
    if len(data) < 20:
        raise OSError("truncated header")
    m, n = (int(x) for x in np.frombuffer(data[4:20], dtype="<u8"))
    if m > (1 << 30) or n > (1 << 30):
        raise OSError("implausible dimensions")
    need = 20 + 8 * m * n
    if len(data) < need:
        raise OSError("truncated header")
    if len(data) > need:
        raise OSError("trailing bytes")
    return np.frombuffer(data[20:need], dtype="<f8").reshape((n, m)).T.copy(order="F")


def lowrank_error(a, t, u, v, k: int, norm: str = "fro") -> float:
    """metrics.cpp:32-46 restated in numpy: ||A - U(:,0:k) T(0:k,:) V'||, Frobenius
    (matrix_ops.cpp:9-14) or the spectral power-iteration estimate (matrix_ops.cpp:16-40)."""
    a, t, u, v = _f(a), _f(t), _f(u), _f(v)
    m, n = a.shape
    if k < 0 or k > min(m, n):
        raise IndexError("lowrank_error: rank out of range")
    e = a - u[:, :k] @ (t[:k, :] @ v.T)
    if norm == "fro":
        return float(np.sqrt(np.sum(e * e)))
    if e.size == 0:
        return 0.0
    x = normal_stream(0x5EEDB0B5, 0, n).reshape(n, 1)
    nx = float(np.sqrt(np.sum(x * x)))
    if nx == 0.0:
        return 0.0
    x /= nx
    est = 0.0
    for it in range(100):
        y = e @ x
        x = e.T @ y
        ny = float(np.sqrt(np.sum(x * x)))
        if ny == 0.0:
            return 0.0
        nxt = float(np.sqrt(ny))
        x /= ny
        if it > 0 and abs(nxt - est) <= 1e-10 * nxt:
            return nxt
        est = nxt
    return est


def optimal_error(sigma, k: int, norm: str = "fro") -> float:
    """metrics.cpp:48-58: sigma_{k+1} (spectral) or sqrt(sum_{i>k} sigma_i^2), summed from the tail."""
    sigma = np.asarray(sigma, dtype=np.float64)
    if k < 0:
        raise IndexError("optimal_error: negative rank")
    if k >= sigma.size:
        return 0.0
    if norm != "fro":
        return float(sigma[k])
    s = 0.0
    for i in range(sigma.size - 1, k - 1, -1):
        s += sigma[i] * sigma[i]
    return float(np.sqrt(s))


def ref_write_rutv(path: str, a) -> None:
    a = _f(a)
    L = _lib("ref")
    L.ref_write_rutv.argtypes = [C.c_char_p, _D, _I64, _I64, _I64]
    rc = L.ref_write_rutv(path.encode(), _p(a), a.shape[0], a.shape[1], max(a.shape[0], 1))
    if rc != 0:
        raise OracleError(rc)


def ref_read_rutv(path: str) -> np.ndarray:
    L = _lib("ref")
    L.ref_read_rutv.argtypes = [C.c_char_p, C.POINTER(_I64), C.POINTER(_I64), _D]
    m, n = _I64(0), _I64(0)
    rc = L.ref_read_rutv(path.encode(), C.byref(m), C.byref(n), None)
    if rc != 0:
        raise OracleError(rc)
    out = np.zeros((m.value, n.value), order="F")
    rc = L.ref_read_rutv(path.encode(), C.byref(m), C.byref(n), _p(out))
    if rc != 0:
        raise OracleError(rc)
    return out


def ref_lowrank_error(a, t, u, v, k: int, norm: str = "fro") -> float:
    a, t, u, v = _f(a), _f(t), _f(u), _f(v)
    L = _lib("ref")
    L.ref_lowrank_error.argtypes = [_D, _D, _D, _D, _I64, _I64, _I64, C.c_int, _D]
    out = C.c_double(0.0)
    rc = L.ref_lowrank_error(_p(a), _p(t), _p(u), _p(v), a.shape[0], a.shape[1], k, int(norm != "fro"),
                             C.byref(out))
    if rc != 0:
        raise OracleError(rc)
    return out.value


def ref_randutv_ab(a, *, b: int, q: int, seed: int, workers: int):
    """The reference's algorithm-by-blocks driver (randutv_ab.hpp:46) on `workers` threads."""
    a = _f(a)
    m, n = a.shape
    L = _lib("ref")
    L.ref_randutv_ab.argtypes = [_D, _I64, _I64, _I64, _I64, C.c_int, C.c_uint64, C.c_int, _D, _D, _D, _D]
    t, u, v = np.zeros((m, n), order="F"), np.zeros((m, m), order="F"), np.zeros((n, n), order="F")
    res = C.c_double(0.0)
    rc = L.ref_randutv_ab(_p(a), m, n, max(m, 1), b, q, seed, workers, _p(t), _p(u), _p(v), C.byref(res))
    if rc != 0:
        raise OracleError(rc, res.value)
    return t, u, v
