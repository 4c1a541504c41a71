"""The C-ABI library: builds, loads, exports every declared symbol (CPU only).

No compute call is made here (there is no GPU in the build container); only
the host-side logic that runs before any device work: option validation with
the reference's ConfigError semantics (randutv_blocked.cpp:10-14), the stream
length and the flop model.
"""
import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle
import paper_2104_05782_b200 as rutv

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    src = open(os.path.join(ROOT, "include", "rutv_b200.h")).read()
    return sorted(set(re.findall(r"\b(rutv_b200_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = rutv.lib()
    syms = _declared_symbols()
    assert len(syms) >= 12
    for s in syms:
        assert hasattr(lib, s), s


def test_library_is_sm100a_only():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", rutv.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_stream_length_and_flops_match_oracle():
    for m, n, b in [(24, 24, 8), (25, 25, 8), (6, 6, 8), (2000, 2000, 128), (4000, 4000, 128),
                    (10000, 10000, 256), (50000, 50000, 512)]:
        assert rutv.stream_length(m, n, b) == oracle.stream_length(m, n, b)
    for n, b, q in [(2000, 128, 0), (4000, 128, 2), (10000, 256, 1), (30000, 256, 2), (50000, 512, 2)]:
        assert rutv.flops(n, b, q) == oracle.flops(n, b, q)


def test_default_opts_mirror_utvconfig():
    o = rutv.Opts()
    rutv.lib().rutv_b200_default_opts(C.byref(o))
    # UTVConfig defaults, randutv_blocked.hpp:11-20
    assert (o.b, o.q, o.build_u, o.build_v, o.seed, o.qr_prepass) == (128, 1, 1, 1, 0, 0)
    assert o.max_steps == -1


@pytest.mark.parametrize("b,q", [(0, 1), (-3, 1), (4, -1)])
def test_config_errors_raise_value_error(b, q):
    a = np.eye(8)
    o = rutv.make_opts(b=max(b, 1), q=q)
    o.b = b
    st = rutv.Status()
    rc = rutv.lib().rutv_b200_factorize(C.byref(o), a.ctypes.data_as(C.c_void_p), 8, 8, 8, None, 0,
                                        a.ctypes.data_as(C.c_void_p), 8, None, 8, None, 8, C.byref(st))
    assert rc == rutv.RUTV_ERR_CONFIG == st.code
    with pytest.raises(ValueError):
        rutv._raise(st)


def test_status_mapping():
    st = rutv.Status()
    st.code, st.residual = rutv.RUTV_ERR_CONVERGENCE, 0.25
    with pytest.raises(rutv.ConvergenceError) as e:
        rutv._raise(st)
    assert e.value.residual == 0.25
    st.code = rutv.RUTV_ERR_INDEX
    with pytest.raises(IndexError):
        rutv._raise(st)


def test_product_does_not_import_oracle():
    """The product package must never route through the CPU oracle."""
    pkg = os.path.join(ROOT, "paper_2104_05782_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f), errors="replace").read()
                assert not re.search(r"^\s*(import|from)\s+oracle", txt, re.M), f
                assert "rutv_oracle" not in txt and "librandutv_ref" not in txt, f


def _build_shim(out):
    import subprocess
    cmd = ["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "shim_example.cpp"),
           "-L", os.path.dirname(rutv.LIB_PATH), "-lrutv_b200",
           f"-Wl,-rpath,{os.path.dirname(rutv.LIB_PATH)}", "-o", out]
    subprocess.run(cmd, check=True, capture_output=True)
    return out


def test_cpp_dropin_header_compiles_and_links(tmp_path):
    """A reference-style C++ caller builds against include/randutv_b200/randutv.hpp
    and links librutv_b200.so (the drop-in of randutv_blocked.hpp:39)."""
    rutv.lib()
    assert os.path.exists(_build_shim(str(tmp_path / "shim")))


def test_grid_local_shape_matches_python_grid():
    """The C++ sharded driver's block-cyclic layout (dist.cu Axis) == dist.Grid
    (block_cyclic.cpp:26-38), including ragged last blocks and ranks that own nothing."""
    from paper_2104_05782_b200.dist import Grid
    for n, b in [(1000, 128), (1024, 128), (50000, 512), (30000, 256), (300, 64), (5, 8), (0, 4)]:
        for P, Q in [(1, 1), (1, 2), (2, 1), (2, 2), (2, 3), (2, 4), (3, 3), (1, 8)]:
            tot_r = tot_c = 0
            for rk in range(P * Q):
                got = rutv.grid_local_shape(n, b, P, Q, rk)
                assert got == Grid(n, b, P, Q, rk).local_shape(), (n, b, P, Q, rk)
                if rk % Q == 0:
                    tot_r += got[0]
                if rk < Q:
                    tot_c += got[1]
            assert tot_r == n and tot_c == n
    with pytest.raises(ValueError):
        rutv.grid_local_shape(100, 8, 2, 2, 4)


def test_opts_grid_fields_default_to_one_gpu():
    o = rutv.make_opts()
    assert (o.grid_p, o.grid_q, o.grid_sim) == (1, 1, 0)
    assert C.sizeof(rutv.Opts) == 72  # the C struct rutv_opts
