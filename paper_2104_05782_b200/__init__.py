"""B200-native blocked randUTV (A = U T V^T) -- Python mirror of the reference API.

The reference exposes ``randutv.factorize(a, *, b=0, q=1, algo="blocked",
workers=1, seed=0, build_uv=True, qr_prepass=False) -> (t, u, v)``
(/root/reference/proj/python/bindings.cpp:49-66, 123-132).  ``factorize`` here
keeps that signature and return convention and adds ``algo="b200"`` (the
default) plus ``g=`` for an explicit Gaussian stream.  It calls the C ABI in
``librutv_b200.so`` (include/rutv_b200.h) -- hand-written sm_100a kernels, no
cuBLAS/cuSOLVER and no CPU fallback: if the library or a GPU is missing the
call raises.

Exception mapping follows bindings.cpp:109-121: ConfigError / ShapeError ->
ValueError, IndexError -> IndexError, ConvergenceError -> ConvergenceError
(a RuntimeError carrying ``.residual``).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "librutv_b200.so")

__all__ = ["factorize", "factorize_device", "flops", "stream_length", "ConvergenceError",
           "RutvError", "lib", "gemm", "hqr", "svd_block", "normal_fill", "apply_q_right",
           "apply_qt_left", "launch_count", "last_profile", "read_rutv", "write_rutv", "lowrank_error",
           "optimal_error", "quality_report", "to_csv"]

RUTV_OK, RUTV_ERR_CONFIG, RUTV_ERR_SHAPE, RUTV_ERR_INDEX, RUTV_ERR_CONVERGENCE = 0, 1, 2, 3, 4
RUTV_ERR_CUDA, RUTV_ERR_NCCL, RUTV_ERR_OOM, RUTV_ERR_NOTIMPL, RUTV_ERR_INTERNAL = 5, 6, 7, 8, 9
RUTV_ERR_IO = 10


class RutvError(RuntimeError):
    def __init__(self, code: int, message: str, residual: float = 0.0):
        super().__init__(message)
        self.code = code
        self.residual = residual


class ConvergenceError(RutvError):
    """Jacobi sweep cap hit (reference ConvergenceError, errors.hpp:29-33)."""


class Status(C.Structure):
    _fields_ = [("code", C.c_int32), ("reserved", C.c_int32), ("residual", C.c_double),
                ("message", C.c_char * 256)]


class Opts(C.Structure):
    _fields_ = [("b", C.c_int64), ("q", C.c_int32), ("build_u", C.c_int32), ("build_v", C.c_int32),
                ("qr_prepass", C.c_int32), ("seed", C.c_uint64), ("device", C.c_int32),
                ("max_steps", C.c_int32), ("overlap", C.c_int32), ("reserved0", C.c_int32),
                ("stream", C.c_uint64), ("grid_p", C.c_int32), ("grid_q", C.c_int32),
                ("grid_sim", C.c_int32), ("keep_workspace", C.c_int32)]


_D = C.POINTER(C.c_double)
_I64 = C.c_int64
_lib = None


def lib() -> C.CDLL:
    """Load librutv_b200.so (building it in place if the sources are newer)."""
    global _lib
    if _lib is not None:
        return _lib
    from . import _build
    if not _build.up_to_date():
        _build.build()
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: the B200 path has no fallback")
    L = C.CDLL(LIB_PATH)
    L.rutv_b200_default_opts.argtypes = [C.POINTER(Opts)]
    L.rutv_b200_stream_length.argtypes = [_I64, _I64, _I64]
    L.rutv_b200_stream_length.restype = _I64
    L.rutv_b200_flops.argtypes = [_I64, _I64, C.c_int32]
    L.rutv_b200_flops.restype = C.c_double
    fac = [C.POINTER(Opts), C.c_void_p, _I64, _I64, _I64, C.c_void_p, _I64, C.c_void_p, _I64,
           C.c_void_p, _I64, C.c_void_p, _I64, C.POINTER(Status)]
    L.rutv_b200_factorize.argtypes = fac
    L.rutv_b200_factorize_device.argtypes = fac
    L.rutv_b200_last_profile.argtypes = [C.POINTER(C.c_char_p), _D, C.c_int]
    L.rutv_b200_launch_count.restype = C.c_uint64
    L.rutv_b200_release_workspace.argtypes = [C.c_int]
    L.rutv_b200_normal_at.argtypes = [C.c_uint64, C.c_uint64]
    L.rutv_b200_normal_at.restype = C.c_double
    L.rutv_b200_build_v_alpha.argtypes = [C.c_int, C.c_void_p, _I64, _I64, _I64, _I64, C.c_int, C.c_uint64,
                                          C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                          C.POINTER(Status)]
    L.rutv_b200_build_u_alpha.argtypes = [C.c_int, C.c_void_p, _I64, _I64, _I64, C.c_void_p, C.c_void_p,
                                          C.c_void_p, C.POINTER(Status)]
    L.rutv_b200_beta_stage.argtypes = [C.c_int, C.c_void_p, _I64, _I64, _I64, _I64, C.c_void_p, C.c_void_p,
                                       C.POINTER(Status)]
    # sharded path (dist.cu)
    L.rutv_b200_grid_local_shape.argtypes = [_I64, _I64, C.c_int, C.c_int, C.c_int, C.POINTER(_I64), C.POINTER(_I64)]
    L.rutv_b200_grid_copy.argtypes = [C.c_int, _I64, _I64, C.c_int, C.c_int, C.c_int, C.c_void_p, _I64, C.c_void_p,
                                      _I64, C.c_int, C.POINTER(Status)]
    L.rutv_b200_nccl_unique_id.argtypes = [C.c_void_p, C.POINTER(Status)]
    L.rutv_b200_dist_create.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p),
                                        C.POINTER(Status)]
    L.rutv_b200_dist_destroy.argtypes = [C.c_void_p, C.POINTER(Status)]
    L.rutv_b200_factorize_dist.argtypes = [C.c_void_p, C.POINTER(Opts), _I64, C.c_void_p, _I64, C.c_void_p, _I64,
                                           C.c_void_p, _I64, C.c_void_p, _I64, C.c_void_p, _I64, C.POINTER(Status)]
    L.rutv_b200_host_alloc.argtypes = [C.c_size_t, C.POINTER(C.c_void_p), C.POINTER(Status)]
    L.rutv_b200_host_free.argtypes = [C.c_void_p, C.POINTER(Status)]
    L.rutv_b200_copy_matrix_async.argtypes = [C.c_void_p, _I64, C.c_void_p, _I64, _I64, _I64, C.c_uint64,
                                              C.POINTER(Status)]
    L.rutv_b200_gemm_profile.argtypes = [_D, _D, C.POINTER(_I64)]
    L.rutv_b200_gaussian_matrix.argtypes = [C.c_int, _I64, _I64, C.c_uint64, C.c_void_p, _I64,
                                            C.POINTER(Status)]
    L.rutv_b200_spectrum_matrix.argtypes = [C.c_int, _I64, _I64, C.c_void_p, C.c_double, C.c_uint64,
                                            C.c_void_p, _I64, C.POINTER(Status)]
    L.rutv_b200_gemm.argtypes = [C.c_int, C.c_double, C.c_int, C.c_void_p, _I64, _I64, _I64, C.c_int,
                                 C.c_void_p, _I64, _I64, _I64, C.c_double, C.c_void_p, _I64, _I64,
                                 _I64, C.POINTER(Status)]
    L.rutv_b200_hqr.argtypes = [C.c_int, C.c_void_p, _I64, _I64, _I64, C.c_void_p, C.c_void_p, _I64,
                                C.POINTER(Status)]
    L.rutv_b200_apply_q_right.argtypes = [C.c_int, C.c_void_p, _I64, _I64, C.c_void_p, _I64, _I64,
                                          C.c_void_p, _I64, _I64, C.POINTER(Status)]
    L.rutv_b200_apply_qt_left.argtypes = L.rutv_b200_apply_q_right.argtypes
    L.rutv_b200_svd_block.argtypes = [C.c_int, C.c_void_p, _I64, _I64, C.c_double, C.c_int,
                                      C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(Status)]
    L.rutv_b200_normal_fill.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_void_p, _I64, _I64,
                                        _I64, C.POINTER(Status)]
    # asynchronous building blocks (dist.py)
    V, S = C.c_void_p, C.POINTER(Status)
    L.rutv_b200_set_stream.argtypes = [C.c_uint64]
    L.rutv_b200_set_stream.restype = None
    L.rutv_b200_gemm_async.argtypes = [C.c_double, C.c_int, V, _I64, _I64, _I64, C.c_int, V, _I64, _I64, _I64,
                                       C.c_double, V, _I64, _I64, _I64, S]
    L.rutv_b200_hqr_async.argtypes = [V, _I64, _I64, _I64, V, S]
    L.rutv_b200_form_wy.argtypes = [V, _I64, _I64, V, _I64, V, _I64, V, _I64, V, _I64, S]
    L.rutv_b200_normal_fill_async.argtypes = [C.c_uint64, C.c_uint64, V, _I64, _I64, _I64, S]
    L.rutv_b200_copy_async.argtypes = [V, _I64, _I64, _I64, V, _I64, S]
    L.rutv_b200_copy_upper_async.argtypes = [V, _I64, _I64, _I64, V, _I64, S]
    L.rutv_b200_identity_async.argtypes = [V, _I64, _I64, _I64, S]
    L.rutv_b200_rect_diag_async.argtypes = [V, _I64, _I64, _I64, V, _I64, S]
    L.rutv_b200_block_rows_async.argtypes = [V, _I64, V, _I64, _I64, _I64, _I64, _I64, _I64, _I64, C.c_int, S]
    L.rutv_b200_svd_batch_async.argtypes = [C.c_int, C.POINTER(_I64), C.POINTER(V), C.POINTER(_I64),
                                            C.POINTER(V), C.POINTER(V), C.POINTER(V), V, S]
    # data format + quality metrics (io_metrics.cu)
    L.rutv_b200_rutv_dims.argtypes = [C.c_char_p, C.POINTER(_I64), C.POINTER(_I64), S]
    L.rutv_b200_read_rutv.argtypes = [C.c_char_p, V, _I64, C.c_int, S]
    L.rutv_b200_write_rutv.argtypes = [C.c_char_p, V, _I64, _I64, _I64, C.c_int, S]
    L.rutv_b200_lowrank_error.argtypes = [C.c_int, V, _I64, V, _I64, V, _I64, V, _I64, _I64, _I64, _I64, C.c_int,
                                          C.c_int, C.c_double, _D, S]
    _lib = L
    return L


def _raise(st: Status) -> None:
    if st.code == RUTV_OK:
        return
    msg = st.message.decode(errors="replace")
    if st.code in (RUTV_ERR_CONFIG, RUTV_ERR_SHAPE):
        raise ValueError(msg)
    if st.code == RUTV_ERR_INDEX:
        raise IndexError(msg)
    if st.code == RUTV_ERR_IO:  # IoError -> OSError (bindings.cpp:109-121)
        raise OSError(msg)
    if st.code == RUTV_ERR_CONVERGENCE:
        raise ConvergenceError(st.code, msg, st.residual)
    raise RutvError(st.code, msg, st.residual)


def make_opts(b: int = 128, q: int = 1, seed: int = 0, build_u: bool = True, build_v: bool = True,
              qr_prepass: bool = False, device: int = 0, max_steps: int = -1,
              overlap: bool = True, stream: int = 0, grid=(1, 1), grid_sim: bool = False,
              keep_workspace: bool = False) -> Opts:
    o = Opts()
    lib().rutv_b200_default_opts(C.byref(o))
    o.grid_p, o.grid_q = int(grid[0]), int(grid[1])
    o.grid_sim = int(grid_sim)
    o.keep_workspace = int(keep_workspace)
    o.b, o.q, o.seed = int(b), int(q), int(seed)
    o.build_u, o.build_v, o.qr_prepass = int(build_u), int(build_v), int(qr_prepass)
    o.device, o.max_steps, o.overlap = int(device), int(max_steps), int(overlap)
    o.stream = int(stream)
    return o


def stream_length(m: int, n: int, b: int) -> int:
    """Gaussian deviates the blocked driver draws (randutv_blocked.cpp:41-44)."""
    return int(lib().rutv_b200_stream_length(m, n, b))


def flops(n: int, b: int, q: int) -> float:
    """Algorithmic flop count F(n, b, q) (U and V built)."""
    return float(lib().rutv_b200_flops(n, b, q))


def _ptr(x: np.ndarray):
    return x.ctypes.data_as(C.c_void_p)


def factorize(a, *, b: int = 0, q: int = 1, algo: str = "b200", seed: int = 0,
              build_uv: bool = True, qr_prepass: bool = False, g=None, device: int = 0,
              max_steps: int = -1, grid=(1, 1), grid_sim: bool = False):
    """Factor ``a`` as ``u @ t @ v.T`` on the B200 (bindings.cpp:49-66 semantics).

    ``g``: optional 1-D array with the first ``stream_length(m, n, b)`` deviates
    of ``RngState(seed)`` -- the bit-identical parity mode; otherwise the sketch
    is drawn on the device from the same counter-based stream.
    ``grid=(P, Q)``: shard over a P x Q block-cyclic grid of GPUs (devices 0 .. P*Q-1, NCCL);
    ``grid_sim=True`` runs the grid's ranks as threads on ``device`` instead (validation).
    Returns ``(t, u, v)``; ``u``/``v`` are None when ``build_uv`` is False."""
    if algo != "b200":
        raise ValueError(f"algo must be 'b200' on this build, got '{algo}'")
    a = np.asfortranarray(np.asarray(a, dtype=np.float64))
    if a.ndim != 2:
        raise ValueError("expected a 2-d array")
    m, n = a.shape
    bb = b if b > 0 else 128
    o = make_opts(b=bb, q=q, seed=seed, build_u=build_uv, build_v=build_uv,
                  qr_prepass=qr_prepass, device=device, max_steps=max_steps, grid=grid, grid_sim=grid_sim)
    t = np.zeros((m, n), order="F")
    u = np.zeros((m, m), order="F") if build_uv else None
    v = np.zeros((n, n), order="F") if build_uv else None
    gp, glen = None, 0
    if g is not None:
        g = np.ascontiguousarray(g, dtype=np.float64)
        gp, glen = _ptr(g), g.size
    st = Status()
    lib().rutv_b200_factorize(C.byref(o), _ptr(a), m, n, max(m, 1), gp, glen, _ptr(t), max(m, 1),
                              _ptr(u) if u is not None else None, max(m, 1),
                              _ptr(v) if v is not None else None, max(n, 1), C.byref(st))
    _raise(st)
    return t, u, v


def factorize_device(a, t, u=None, v=None, *, b: int = 128, q: int = 1, seed: int = 0,
                     g=None, device: int | None = None, max_steps: int = -1,
                     stream: int = 0, qr_prepass: bool = False) -> None:
    """Device-resident variant on torch CUDA tensors (column-major = a
    transposed contiguous row-major tensor; pass ``x.T`` views with stride (1, ld))."""
    def info(x):
        if x is None:
            return None, 1
        assert x.dtype.itemsize == 8 and x.stride(0) == 1, "column-major fp64 tensor expected"
        return C.c_void_p(x.data_ptr()), max(x.stride(1), x.shape[0], 1)
    m, n = a.shape
    dev = a.device.index if device is None else device
    o = make_opts(b=b, q=q, seed=seed, build_u=u is not None, build_v=v is not None, device=dev,
                  max_steps=max_steps, stream=stream, qr_prepass=qr_prepass)
    pa, lda = info(a)
    pt, ldt = info(t)
    pu, ldu = info(u)
    pv, ldv = info(v)
    gp, glen = (C.c_void_p(g.data_ptr()), g.numel()) if g is not None else (None, 0)
    st = Status()
    lib().rutv_b200_factorize_device(C.byref(o), pa, m, n, lda, gp, glen, pt, ldt, pu, ldu, pv, ldv,
                                     C.byref(st))
    _raise(st)


class PinnedMatrix:
    """Page-locked host matrix of exactly m x n doubles (column-major), allocated
    with ``rutv_b200_host_alloc``; ``.array`` is a Fortran-ordered numpy view.
    Free with ``close()`` (or let it be garbage collected)."""

    def __init__(self, m: int, n: int):
        self.ptr = C.c_void_p()
        st = Status()
        lib().rutv_b200_host_alloc(max(m * n, 1) * 8, C.byref(self.ptr), C.byref(st))
        _raise(st)
        buf = (C.c_double * max(m * n, 1)).from_address(self.ptr.value)
        self.array = np.frombuffer(buf, dtype=np.float64, count=m * n).reshape((n, m)).T
        self.shape = (m, n)

    def close(self) -> None:
        if self.ptr is not None and self.ptr.value:
            self.array = None
            st = Status()
            lib().rutv_b200_host_free(self.ptr, C.byref(st))
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------- the reference's public step API (randutv_blocked.hpp:41-72) ----------------
def normal_at(seed: int, d: int) -> float:
    """RngState(seed).normal_at(d) on the host (rng.cpp:29-36)."""
    return float(lib().rutv_b200_normal_at(seed, d))


def build_v_alpha(t22, b: int, q: int, seed: int, pos: int, g=None, device: int = 0):
    """build_v_alpha (randutv_blocked.cpp:40-55) on the B200: returns (qr, tau, twy) of the
    QR of Y = (T22' T22)^q T22' G, G = deviates pos .. pos + rows*b of RngState(seed)
    (device-drawn) or the explicit ``g`` (rows x b, the bit-identical parity mode).  The
    caller advances its position by rows*b, as the reference's RngState& does."""
    t22 = np.asfortranarray(np.asarray(t22, dtype=np.float64))
    rows, cols = t22.shape
    p = min(cols, b)
    qr = np.zeros((cols, b), order="F")
    tau = np.zeros(max(p, 1))
    twy = np.zeros((p, p), order="F")
    gp = None
    if g is not None:
        g = np.asfortranarray(np.asarray(g, dtype=np.float64).reshape((rows, b), order="F"))
        gp = _ptr(g)
    st = Status()
    lib().rutv_b200_build_v_alpha(device, _ptr(t22), rows, cols, max(rows, 1), b, q, seed, pos, gp, _ptr(qr),
                                  _ptr(tau), _ptr(twy), C.byref(st))
    _raise(st)
    return qr, tau[:p], twy


def build_u_alpha(panel, device: int = 0):
    """build_u_alpha (randutv_blocked.cpp:57-63): ``panel`` (Fortran float64) is factored
    in place; returns (qr copy, tau, twy)."""
    if not (isinstance(panel, np.ndarray) and panel.dtype == np.float64 and panel.flags.f_contiguous):
        raise ValueError("build_u_alpha works in place on a Fortran-ordered float64 array")
    rows, cols = panel.shape
    p = min(rows, cols)
    qr = np.zeros((rows, cols), order="F")
    tau = np.zeros(max(p, 1))
    twy = np.zeros((p, p), order="F")
    st = Status()
    lib().rutv_b200_build_u_alpha(device, _ptr(panel), rows, cols, max(rows, 1), _ptr(qr), _ptr(tau), _ptr(twy),
                                  C.byref(st))
    _raise(st)
    return qr, tau[:p], twy


def beta_stage(t22, bw: int, device: int = 0):
    """beta_stage (randutv_blocked.cpp:65-81): ``t22`` (Fortran float64) updated in place;
    returns (u rt x rt, v bw x bw)."""
    if not (isinstance(t22, np.ndarray) and t22.dtype == np.float64 and t22.flags.f_contiguous):
        raise ValueError("beta_stage works in place on a Fortran-ordered float64 array")
    rows, cols = t22.shape
    rt = min(rows, bw)
    u = np.zeros((max(rt, 0), max(rt, 0)), order="F")
    v = np.zeros((max(bw, 0), max(bw, 0)), order="F")
    st = Status()
    lib().rutv_b200_beta_stage(device, _ptr(t22), rows, cols, max(rows, 1), bw, _ptr(u) if u.size else None,
                               _ptr(v) if v.size else None, C.byref(st))
    _raise(st)
    return u, v


# ---------------- sharded path: one process per GPU (dist.cu) ----------------
def grid_local_shape(n: int, b: int, P: int, Q: int, rank: int) -> tuple[int, int]:
    """(local rows, local cols) of ``rank`` on the P x Q block-cyclic grid (block_cyclic.cpp:26-38)."""
    r, c = _I64(0), _I64(0)
    if lib().rutv_b200_grid_local_shape(n, b, P, Q, rank, C.byref(r), C.byref(c)) != RUTV_OK:
        raise ValueError("bad grid")
    return r.value, c.value


def grid_copy(full, loc, n: int, b: int, P: int, Q: int, rank: int, to_local: bool) -> None:
    """Full n x n column-major CUDA tensor <-> this rank's local blocks (column-major CUDA tensor)."""
    pf, _, _, ldf = _cm(full)
    pl, _, _, ldl = _cm(loc)
    st = Status()
    lib().rutv_b200_grid_copy(loc.device.index or 0, n, b, P, Q, rank, pf, ldf, pl, ldl, int(to_local), C.byref(st))
    _raise(st)


def nccl_unique_id() -> bytes:
    buf = (C.c_ubyte * 128)()
    st = Status()
    lib().rutv_b200_nccl_unique_id(buf, C.byref(st))
    _raise(st)
    return bytes(buf)


class DistContext:
    """One rank of a P x Q grid (its NCCL communicators); collective to create."""

    def __init__(self, uid: bytes, P: int, Q: int, rank: int, device: int):
        self.P, self.Q, self.rank, self.device = P, Q, rank, device
        self.h = C.c_void_p()
        idb = (C.c_ubyte * 128).from_buffer_copy(uid)
        st = Status()
        lib().rutv_b200_dist_create(idb, P, Q, rank, device, C.byref(self.h), C.byref(st))
        _raise(st)

    def close(self) -> None:
        if self.h is not None and self.h.value:
            st = Status()
            lib().rutv_b200_dist_destroy(self.h, C.byref(st))
            self.h = None

    def factorize(self, n: int, a_loc, t_loc, u_loc=None, v_loc=None, *, b: int = 128, q: int = 1, seed: int = 0,
                  g=None, stream: int = 0, max_steps: int = -1, overlap: bool = True) -> None:
        """This rank's part of the sharded factorization (column-major CUDA tensors: A, T, U, V
        local blocks; in place when v_loc sits directly on top of t_loc in one buffer)."""
        def info(x):
            if x is None:
                return None, 1
            return C.c_void_p(x.data_ptr()), max(x.stride(1) if x.shape[1] > 1 else x.shape[0], x.shape[0], 1)
        o = make_opts(b=b, q=q, seed=seed, build_u=u_loc is not None, build_v=v_loc is not None,
                      device=self.device, max_steps=max_steps, overlap=overlap, stream=stream)
        pa, lda = info(a_loc)
        pt, ldt = info(t_loc)
        pu, ldu = info(u_loc)
        pv, ldv = info(v_loc)
        gp, glen = (C.c_void_p(g.data_ptr()), g.numel()) if g is not None else (None, 0)
        st = Status()
        lib().rutv_b200_factorize_dist(self.h, C.byref(o), n, pa, lda, gp, glen, pt, ldt, pu, ldu, pv, ldv,
                                       C.byref(st))
        _raise(st)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _mat_ptr(x):
    """(pointer, rows, cols, ld) of a column-major FP64 matrix: a Fortran-ordered numpy array
    (e.g. PinnedMatrix.array) or a column-major torch tensor (stride (1, ld))."""
    if isinstance(x, np.ndarray):
        assert x.dtype == np.float64 and x.strides[0] == 8, "column-major float64 array expected"
        r, c = x.shape
        return C.c_void_p(x.ctypes.data), r, c, max(x.strides[1] // 8 if c > 1 else r, r, 1)
    assert x.dtype.itemsize == 8 and (x.stride(0) == 1 or x.numel() == 0), "column-major fp64 tensor expected"
    r, c = x.shape
    return C.c_void_p(x.data_ptr()), r, c, max(x.stride(1) if c > 1 else r, r, 1)


def copy_matrix_async(dst, src, stream: int = 0) -> None:
    """dst <- src between host and device memory (rutv_b200_copy_matrix_async), async on ``stream``."""
    pd, r, c, ldd = _mat_ptr(dst)
    ps, r2, c2, lds = _mat_ptr(src)
    if (r, c) != (r2, c2):
        raise ValueError("copy_matrix_async: shape mismatch")
    st = Status()
    lib().rutv_b200_copy_matrix_async(pd, ldd, ps, lds, r, c, stream, C.byref(st))
    _raise(st)


def release_workspace(device: int = 0) -> None:
    """Return the library pool's cached device memory (kept by keep_workspace calls)."""
    lib().rutv_b200_release_workspace(device)


def launch_count() -> int:
    return int(lib().rutv_b200_launch_count())


def last_profile() -> dict:
    names = (C.c_char_p * 16)()
    ms = (C.c_double * 16)()
    k = lib().rutv_b200_last_profile(names, ms, 16)
    return {names[i].decode(): ms[i] for i in range(k)}


# ---------------- L1 kernels on torch CUDA tensors (column-major views) ----------------

def _cm(x):
    """(ptr, rows, cols, ld) of a column-major fp64 CUDA tensor view (stride(0) == 1)."""
    assert x.is_cuda and x.stride(0) == 1 or x.numel() == 0, "column-major CUDA tensor expected"
    r, c = x.shape
    return C.c_void_p(x.data_ptr()), r, c, max(x.stride(1) if c > 1 else r, r, 1)


def gemm(alpha, ta, a, tb, b, beta, c) -> None:
    """In-place ``c <- alpha op(a) op(b) + beta c`` (proj/src/gemm.cpp:21)."""
    pa, ar, ac, lda = _cm(a)
    pb, br, bc, ldb = _cm(b)
    pc, m, n, ldc = _cm(c)
    st = Status()
    lib().rutv_b200_gemm(c.device.index, alpha, int(ta), pa, ar, ac, lda, int(tb), pb, br, bc, ldb,
                         beta, pc, m, n, ldc, C.byref(st))
    _raise(st)


def hqr(a, tau, twy) -> None:
    """In-place packed QR + Twy (householder.cpp:48-97)."""
    pa, m, n, lda = _cm(a)
    pt, p, _, ldt = _cm(twy)
    st = Status()
    lib().rutv_b200_hqr(a.device.index, pa, m, n, lda, C.c_void_p(tau.data_ptr()), pt, ldt,
                        C.byref(st))
    _raise(st)


def apply_q_right(qr, twy, bmat) -> None:
    pq, s, p, ldq = _cm(qr)
    pt, _, _, ldt = _cm(twy)
    pb, rows, _, ldb = _cm(bmat)
    st = Status()
    lib().rutv_b200_apply_q_right(bmat.device.index, pq, s, ldq, pt, twy.shape[0], ldt, pb, rows, ldb,
                                  C.byref(st))
    _raise(st)


def apply_qt_left(qr, twy, bmat) -> None:
    pq, s, p, ldq = _cm(qr)
    pt, _, _, ldt = _cm(twy)
    pb, _, cols, ldb = _cm(bmat)
    st = Status()
    lib().rutv_b200_apply_qt_left(bmat.device.index, pq, s, ldq, pt, twy.shape[0], ldt, pb, cols,
                                  ldb, C.byref(st))
    _raise(st)


def svd_block(a, u, sigma, v, tol: float = 1e-15, max_sweeps: int = 30) -> None:
    pa, n, _, lda = _cm(a)
    st = Status()
    lib().rutv_b200_svd_block(a.device.index, pa, n, lda, tol, max_sweeps, C.c_void_p(u.data_ptr()),
                              C.c_void_p(sigma.data_ptr()), C.c_void_p(v.data_ptr()), C.byref(st))
    _raise(st)


def normal_fill(seed: int, pos: int, g) -> None:
    pg, r, c, ld = _cm(g)
    st = Status()
    lib().rutv_b200_normal_fill(g.device.index, seed, pos, pg, r, c, ld, C.byref(st))
    _raise(st)


def gemm_profile() -> dict:
    """GEMM totals of the last factorize call (needs RUTV_GEMM_PROFILE=1)."""
    f, ms, n = C.c_double(), C.c_double(), _I64()
    lib().rutv_b200_gemm_profile(C.byref(f), C.byref(ms), C.byref(n))
    return {"flops": f.value, "ms": ms.value, "launches": n.value}


def gaussian_matrix_device(a, seed: int) -> None:
    """gaussian_matrix (metrics.cpp:90-93) into a column-major CUDA tensor."""
    pa, m, n, lda = _cm(a)
    st = Status()
    lib().rutv_b200_gaussian_matrix(a.device.index, m, n, seed, pa, lda, C.byref(st))
    _raise(st)


def spectrum_matrix_device(a, seed: int, sigma=None, beta: float = 1.0) -> None:
    """Q1 diag(sigma) Q2^T with Haar factors (metrics.cpp:24-28, 95-110) on the device;
    sigma=None gives geometric_matrix's beta^j."""
    pa, m, n, lda = _cm(a)
    sp = None
    if sigma is not None:
        sigma = np.ascontiguousarray(sigma, dtype=np.float64)
        sp = _ptr(sigma)
    st = Status()
    lib().rutv_b200_spectrum_matrix(a.device.index, m, n, sp, beta, seed, pa, lda, C.byref(st))
    _raise(st)


# ----------------------------------------------------------------- data format + metrics
def _is_cuda(x) -> bool:
    return hasattr(x, "is_cuda") and x.is_cuda


def write_rutv(path: str, a) -> None:
    """randutv::write_rutv (proj/src/matrix_io.cpp:40-50) from a host array or a CUDA
    tensor (column-major or any 2-D layout; device tensors stream through pinned buffers)."""
    st = Status()
    if _is_cuda(a):
        x = a if a.stride(0) == 1 else a.T.contiguous().T  # column-major view
        ld = max(x.stride(1) if x.shape[1] > 1 else x.shape[0], x.shape[0], 1)
        lib().rutv_b200_write_rutv(os.fsencode(path), C.c_void_p(x.data_ptr()), x.shape[0], x.shape[1], ld, 1,
                                   C.byref(st))
    else:
        x = np.asfortranarray(np.asarray(a, dtype=np.float64))
        lib().rutv_b200_write_rutv(os.fsencode(path), _ptr(x), x.shape[0], x.shape[1], max(x.shape[0], 1), 0,
                                   C.byref(st))
    _raise(st)


def read_rutv(path: str, device=None):
    """randutv::read_rutv (proj/src/matrix_io.cpp:52-70).  ``device=None``: a Fortran-ordered
    numpy array; else a column-major CUDA tensor on that device (payload streamed to HBM)."""
    st = Status()
    m, n = _I64(0), _I64(0)
    lib().rutv_b200_rutv_dims(os.fsencode(path), C.byref(m), C.byref(n), C.byref(st))
    _raise(st)
    m, n = m.value, n.value
    if device is None:
        out = np.zeros((m, n), order="F")
        lib().rutv_b200_read_rutv(os.fsencode(path), _ptr(out), max(m, 1), 0, C.byref(st))
    else:
        import torch
        out = torch.empty((n, m), dtype=torch.float64, device=device).T
        lib().rutv_b200_read_rutv(os.fsencode(path), C.c_void_p(out.data_ptr()), max(m, 1), 1, C.byref(st))
    _raise(st)
    return out


def lowrank_error(a, t, u, v, k: int, norm: str = "fro") -> float:
    """randutv::lowrank_error (proj/src/metrics.cpp:32-46) on the device: CUDA tensors
    A (m x n), T (m x n), U (m x m), V (n x n); norm "fro" or "spectral"."""
    st = Status()
    out = C.c_double(0.0)
    pa, pt, pu, pv = (_cm(x) for x in (a, t, u, v))
    m, n = a.shape
    if t.shape != (m, n) or u.shape != (m, m) or v.shape != (n, n):
        raise ValueError("lowrank_error: needs square U and V matching A")
    lib().rutv_b200_lowrank_error(a.device.index or 0, pa[0], pa[3], pt[0], pt[3], pu[0], pu[3], pv[0], pv[3], m, n,
                                  int(k), 0 if norm == "fro" else 1, 0, 0.0, C.byref(out), C.byref(st))
    _raise(st)
    return out.value


def optimal_error(sigma, k: int, norm: str = "fro") -> float:
    """randutv::optimal_error (metrics.cpp:48-58) from known singular values."""
    sig = np.asarray(sigma, dtype=np.float64)
    if k < 0:
        raise IndexError("optimal_error: negative rank")
    if k >= sig.size:
        return 0.0
    if norm != "fro":
        return float(sig[k])
    tail = sig[k:][::-1]
    return float(np.sqrt(np.sum(tail * tail)))


def quality_report(a, t, u, v, ks, sigma, norm: str = "fro") -> list[dict]:
    """randutv::quality_report (metrics.cpp:161-184) with the residuals on the device.
    ``sigma``: the singular values of A (known by construction for the spectrum
    generators; the reference computes them with a dense Jacobi SVD)."""
    p = min(a.shape)
    sig = np.asarray(sigma, dtype=np.float64)
    diag = t.diagonal().double().cpu().numpy() if _is_cuda(t) else np.diag(t)
    rows = []
    for k in ks:
        if k < 1 or k > p:
            raise IndexError("quality_report: ranks must satisfy 1 <= k <= min(m, n)")
        e_utv = lowrank_error(a, t, u, v, k, norm)
        e_opt = optimal_error(sig, k, norm)
        ratio = e_utv / e_opt if e_opt > 0 else (1.0 if e_utv == 0 else float("inf"))
        s, d = sig[k - 1], diag[k - 1]
        rows.append({"k": int(k), "err_utv": e_utv, "err_opt": e_opt, "ratio": ratio,
                     "diag_relerr": abs(d - s) / s if s > 0 else abs(d)})
    return rows


def to_csv(rows: list[dict]) -> str:
    """metrics.cpp:186-197: header k,err_utv,err_opt,ratio,diag_relerr, %.17g values."""
    out = ["k,err_utv,err_opt,ratio,diag_relerr"]
    for r in rows:
        out.append("%d,%s,%s,%s,%s" % (r["k"], *("%.17g" % r[c] for c in ("err_utv", "err_opt", "ratio", "diag_relerr"))))
    return "\n".join(out) + "\n"
